// jit.cu — weight-specialised SpMM kernels (NVRTC, compiled on first use).
//
// The tile kernel (spmm_kernel.cuh) is bound by its shared-memory gather: one
// activation load per stored weight per column. Here the sparse structure and
// the weights are compiled into the instruction stream instead:
//
//  * k-major order. A warp owns a group of 64 virtual columns (2 per lane,
//    f32x2 registers) and keeps one accumulator pair per output row of its
//    row segment in registers. Activation rows stream through shared memory
//    in chunks of 32 channels (cp.async, P-deep ring per warp); each channel
//    pair is loaded once (LDS.64) and feeds every row of the segment that
//    stores a block at that channel, as FMUL2-with-immediate + FFMA2 (strict)
//    or FFMA2-with-immediate (fast). Per row the terms still arrive in
//    ascending channel order after the bias (kernels.cpp:14-43), so strict
//    mode is bit-exact: fma.rn.f32x2(acc, 1.0, p) rounds acc + p once, exactly
//    like add.rn (the 1.0 is a kernel argument so ptxas cannot fold the pair
//    back into a fused multiply-add).
//
//  * Row segments across SMs. Straight-line code only runs at full rate while
//    it fits the SM's instruction cache, so the rows are cut into segments of
//    at most ~kJitSegInstr instructions and one persistent CTA per SM runs one
//    segment; SMs are shared out in proportion to segment cost. The segments
//    sweep the column groups in the same order at the same rate, so the
//    activations each group needs are read from HBM once and served to the
//    other segments from L2.
//
// Clamp is the ternary compare of Activation::apply (tensor.hpp:90-96), done
// per column on the unpacked pair. Rows >= m_out (padding of a model layer,
// netdef.cpp:496-505) are not generated. Requires S % 4 == 0 and 16 B aligned
// activations (key.vec); other shapes use the tile kernel.
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "spcv_internal.h"

using namespace spcv_detail;

namespace {

constexpr int kKC = 32;        // channels per staged chunk
constexpr int kRowsMax = 128;  // rows per segment

// Rows a segment may hold so that its accumulators (cpl registers per row:
// columns per lane) fit the register budget of a W-warp CTA (65536 / (32 W),
// at most 255) with ~48 to spare.
int rows_max(int warps, int cpl) {
    const int regs = std::min(255, 65536 / (32 * warps));
    return std::max(8, std::min(kRowsMax / cpl, (regs - 48) / cpl));
}

int knob(int v, int dflt) { return v > 0 ? v : dflt; }

// f32 bit pattern duplicated into both halves of a .b64 (f32x2 broadcast).
std::string imm2(float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    char buf[40];
    std::snprintf(buf, sizeof buf, "0x%08x%08xULL", u, u);
    return buf;
}

struct Segment {
    int r0 = 0, r1 = 0;      // stored rows [r0, r1)
    long long instr = 0;     // straight-line instructions per column group
    int ctas = 0;
};

int row_nnz(const uint32_t* row_ptr, int BH, int r) {
    return static_cast<int>(row_ptr[r / BH + 1] - row_ptr[r / BH]);
}

// Cut rows [0, m_out) into segments (contiguous rows, cost <= budget, at most
// kRowsMax rows) and share `sms` CTAs out in proportion to their cost.
bool plan_segments(int M, int K, int BH, const uint32_t* row_ptr, const JitKey& key, const Knobs& kn,
                   std::vector<Segment>& segs) {
    const int budget = knob(kn.jit_seg_instr, kJitSegInstr);
    const int max_segs = std::min(knob(kn.jit_max_segs, kJitMaxSegs), key.sms);
    const int per_weight = key.strict ? 2 : 1;
    const int nkc = (K + kKC - 1) / kKC;
    const long long fixed = static_cast<long long>(nkc) * 24 + K;  // copies, waits, LDS.64
    const int rows = std::min(M, key.m_out);
    segs.clear();
    Segment cur;
    cur.instr = fixed;
    for (int r = 0; r < rows; ++r) {
        const long long c = static_cast<long long>(per_weight) * row_nnz(row_ptr, BH, r) + 10;
        if (cur.r1 > cur.r0 && (cur.instr + c > budget || cur.r1 - cur.r0 == rows_max(key.warps, key.cpl))) {
            segs.push_back(cur);
            cur = Segment();
            cur.r0 = cur.r1 = r;
            cur.instr = fixed;
        }
        cur.r1 = r + 1;
        cur.instr += c;
    }
    if (cur.r1 > cur.r0) segs.push_back(cur);
    if (segs.empty() || static_cast<int>(segs.size()) > max_segs) return false;
    long long total = 0;
    for (const Segment& s : segs) total += s.instr;
    int given = 0;
    for (Segment& s : segs) {
        s.ctas = std::max(1, static_cast<int>(static_cast<double>(key.sms) * s.instr / total));
        given += s.ctas;
    }
    // hand out the remainder / take back the excess by cost per CTA
    while (given != key.sms) {
        int best = -1;
        double bv = 0;
        for (size_t i = 0; i < segs.size(); ++i) {
            const double load = static_cast<double>(segs[i].instr) / segs[i].ctas;
            if (given < key.sms) {
                if (best < 0 || load > bv) best = static_cast<int>(i), bv = load;
            } else if (segs[i].ctas > 1) {
                const double after = static_cast<double>(segs[i].instr) / (segs[i].ctas - 1);
                if (best < 0 || after < bv) best = static_cast<int>(i), bv = after;
            }
        }
        if (best < 0) return false;
        segs[best].ctas += given < key.sms ? 1 : -1;
        given += given < key.sms ? 1 : -1;
    }
    return true;
}

std::string gen_source(int M, int K, int BH, const uint32_t* row_ptr, const uint32_t* col_idx,
                       const float* values, const JitKey& key, const Knobs& kn, const std::vector<Segment>& segs) {
    const int nkc = (K + kKC - 1) / kKC;
    const int C = key.cpl;             // columns per lane: 2 (f32x2) or 1 (scalar)
    const int kCols = 32 * C;          // columns per warp group
    const int Q = kCols / 4;           // 16 B quads per staged channel row
    const int RPI = 32 / Q;            // channel rows one warp-wide copy covers
    std::ostringstream o;
    o << "#define K " << K << "LL\n#define KC " << kKC << "\n#define NKC " << nkc
      << "\n#define W " << key.warps << "\n#define P " << key.stages << "\n"
      << "typedef unsigned long long u64;\n"
      << "__device__ __forceinline__ unsigned sa(const void* p) {"
         " return (unsigned)__cvta_generic_to_shared(p); }\n"
      << "#define CP16(d, off, s) asm volatile(\"cp.async.cg.shared.global [%0+\" #off \"], [%1], 16;\" :: \"r\"(d), \"l\"(s) : \"memory\")\n"
      << "#define LDS64(v, a, off) asm volatile(\"ld.shared.b64 %0, [%1+\" #off \"];\" : \"=l\"(v) : \"r\"(a))\n"
      << "#define LDS32(v, a, off) asm volatile(\"ld.shared.f32 %0, [%1+\" #off \"];\" : \"=f\"(v) : \"r\"(a))\n"
      << "__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 d;"
         " asm(\"mul.rn.f32x2 %0, %1, %2;\" : \"=l\"(d) : \"l\"(a), \"l\"(b)); return d; }\n"
      << "__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d;"
         " asm(\"fma.rn.f32x2 %0, %1, %2, %3;\" : \"=l\"(d) : \"l\"(a), \"l\"(b), \"l\"(c)); return d; }\n"
      << "__device__ __forceinline__ u64 dup(float f) {"
         " return ((u64)__float_as_uint(f) << 32) | __float_as_uint(f); }\n"
      << "__device__ __forceinline__ float lo32(u64 v) { return __uint_as_float((unsigned)v); }\n"
      << "__device__ __forceinline__ float hi32(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }\n"
      << "__device__ __forceinline__ float clampf(float v, float lo, float hi) {"
         " return v < lo ? lo : (v > hi ? hi : v); }\n";
    // CTA -> (segment, rank in segment), segments interleaved round-robin so
    // neighbouring CTAs (and both dies) run every segment
    std::vector<int> seg_of, rank_of, left;
    for (const Segment& sg : segs) left.push_back(sg.ctas);
    for (bool any = true; any;) {
        any = false;
        for (size_t s = 0; s < segs.size(); ++s)
            if (left[s] > 0) {
                seg_of.push_back(static_cast<int>(s));
                rank_of.push_back(segs[s].ctas - left[s]);
                --left[s];
                any = true;
            }
    }
    if (kn.jit_interleave == 0) {
        seg_of.clear();
        rank_of.clear();
        for (size_t s = 0; s < segs.size(); ++s)
            for (int c = 0; c < segs[s].ctas; ++c) seg_of.push_back(static_cast<int>(s)), rank_of.push_back(c);
    }
    o << "__device__ const unsigned char seg_of[" << key.sms << "] = {";
    for (int v : seg_of) o << v << ",";
    o << "};\n__device__ const unsigned char rank_of[" << key.sms << "] = {";
    for (int v : rank_of) o << v << ",";
    o << "};\n";

    const int brows = M / BH;
    std::vector<std::vector<std::pair<int, float>>> by_k;  // (row in segment, weight) per channel
    for (size_t si = 0; si < segs.size(); ++si) {
        const Segment& sg = segs[si];
        const int R = sg.r1 - sg.r0;
        by_k.assign(static_cast<size_t>(K), {});
        for (int r = sg.r0; r < sg.r1; ++r) {
            const int br = r / BH, i = r % BH;
            if (br >= brows) continue;
            for (uint32_t b = row_ptr[br]; b < row_ptr[br + 1]; ++b)
                by_k[col_idx[b]].emplace_back(r - sg.r0, values[static_cast<size_t>(b) * BH + i]);
        }
        o << "__device__ __forceinline__ void seg" << si
          << "(const float* __restrict__ act, float* __restrict__ out, const float* __restrict__ bias,"
             " long long N, long long S, float lo, float hi, const float* __restrict__ res, u64 one,"
             " float* ring, int lane, long long first, long long stride) {\n"
          << "  const long long G = (N + " << kCols - 1 << ") / " << kCols << ";\n"
          << "  const long long ng = first < G ? (G - first + stride - 1) / stride : 0;\n"
          << "  long long ig = 0; int ikc = 0; bool valid = false; const float* src = nullptr;\n"
          << "  auto set_src = [&](long long gi) {\n"
          << "    const long long nq = (first + gi * stride) * " << kCols << " + 4 * (lane % " << Q << ");\n"
          << "    valid = gi < ng && nq < N;\n"
          << "    if (valid) { const long long b = nq / S, s = nq - b * S;"
             " src = act + b * K * S + s + (lane / " << Q << ") * S; }\n"
          << "  };\n"
          << "  const unsigned ring_sa = sa(ring);\n"
          << "  int islot = 0, cslot = 0;\n"
          << "  auto issue = [&]() {\n"
          << "    const unsigned dst = ring_sa + islot * (KC * " << kCols * 4 << ") + ((lane / " << Q << ") * "
          << kCols << " + 4 * (lane % " << Q << ")) * 4;\n"
          << "    if (valid) {\n"
          << "      const float* sk = src + (long long)ikc * KC * S;\n";
        for (int j = 0; j < kKC / RPI; ++j) {
            const std::string cp = "CP16(dst, " + std::to_string(RPI * j * kCols * 4) + ", sk + " +
                                   std::to_string(RPI * j) + "LL * S);";
            if (K % kKC == 0)
                o << "      " << cp << "\n";
            else
                o << "      if (ikc * KC + (lane / " << Q << ") + " << RPI * j << " < K) " << cp << "\n";
        }
        o << "    }\n"
          << "    asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n"
          << "    if (++islot == P) islot = 0;\n"
          << "    if (++ikc == NKC) { ikc = 0; ++ig; set_src(ig); }\n"
          << "  };\n"
          << "  set_src(0);\n"
          << "#pragma unroll 1\n"
          << "  for (int p = 0; p < P - 1; ++p) issue();\n"
          << "#pragma unroll 1\n"
          << "  for (long long gi = 0; gi < ng; ++gi) {\n";
        for (int q = 0; q < R; ++q) {
            const int r = sg.r0 + q;
            if (C == 2)
                o << "    u64 a" << q << " = " << (key.bias ? "dup(__ldg(bias + " + std::to_string(r) + "))" : "0ULL")
                  << ";\n";
            else
                o << "    float a" << q << " = " << (key.bias ? "__ldg(bias + " + std::to_string(r) + ")" : "0.0f")
                  << ";\n";
        }
        for (int kc = 0; kc < nkc; ++kc) {
            o << "    issue();\n"
              << "    asm volatile(\"cp.async.wait_group %0;\" :: \"n\"(P - 1) : \"memory\");\n"
              << "    __syncwarp();\n"
              << "    { const unsigned xs = ring_sa + cslot * (KC * " << kCols * 4 << ") + " << 4 * C
              << " * lane;\n";
            for (int k = kc * kKC; k < std::min(K, (kc + 1) * kKC); ++k) {
                if (by_k[k].empty()) continue;
                if (C == 2)
                    o << "      { u64 x; LDS64(x, xs, " << (k - kc * kKC) * kCols * 4 << ");\n";
                else
                    o << "      { float x; LDS32(x, xs, " << (k - kc * kKC) * kCols * 4 << ");\n";
                for (const auto& [q, v] : by_k[k]) {
                    if (C == 1) {
                        uint32_t u;
                        std::memcpy(&u, &v, 4);
                        char wv[40];
                        std::snprintf(wv, sizeof wv, "__uint_as_float(0x%08xu)", u);
                        if (key.strict)
                            o << "        a" << q << " = __fadd_rn(a" << q << ", __fmul_rn(" << wv << ", x));\n";
                        else
                            o << "        a" << q << " = __fmaf_rn(" << wv << ", x, a" << q << ");\n";
                    } else if (key.strict) {
                        o << "        a" << q << " = fma2(a" << q << ", one, mul2(" << imm2(v) << ", x));\n";
                    } else {
                        o << "        a" << q << " = fma2(" << imm2(v) << ", x, a" << q << ");\n";
                    }
                }
                o << "      }\n";
            }
            o << "    }\n    __syncwarp();\n    if (++cslot == P) cslot = 0;\n";
        }
        if (C == 2) {
        o << "    const long long n0 = (first + gi * stride) * " << kCols << " + 2 * lane;\n"
          << "    if (n0 < N) {\n"
          << "      const long long b = n0 / S, s = n0 - b * S;\n"
          << "      const int S2 = (int)(S >> 1);\n"
          << "      float2* op = reinterpret_cast<float2*>(out + (b * " << key.m_out << "LL + " << sg.r0
          << ") * S + s);\n";
        if (key.res)
            o << "      const float2* rp = reinterpret_cast<const float2*>(res + (b * " << key.m_out
              << "LL + " << sg.r0 << ") * S + s);\n";
        for (int q = 0; q < R; ++q) {
            o << "      { float2 v = make_float2(lo32(a" << q << "), hi32(a" << q << "));\n";
            if (key.clamp) o << "        v.x = clampf(v.x, lo, hi); v.y = clampf(v.y, lo, hi);\n";
            if (key.res)
                o << "        { const float2 t = __ldcs(rp); rp += S2;"
                     " v.x = __fadd_rn(v.x, t.x); v.y = __fadd_rn(v.y, t.y); }\n";
            o << "        __stcs(op, v); op += S2; }  // row " << sg.r0 + q << "\n";
        }
        } else {
        o << "    const long long n0 = (first + gi * stride) * " << kCols << " + lane;\n"
          << "    if (n0 < N) {\n"
          << "      const long long b = n0 / S, s = n0 - b * S;\n"
          << "      const int S1 = (int)S;\n"
          << "      float* op = out + (b * " << key.m_out << "LL + " << sg.r0 << ") * S + s;\n";
        if (key.res)
            o << "      const float* rp = res + (b * " << key.m_out << "LL + " << sg.r0 << ") * S + s;\n";
        for (int q = 0; q < R; ++q) {
            o << "      { float v = a" << q << ";\n";
            if (key.clamp) o << "        v = clampf(v, lo, hi);\n";
            if (key.res) o << "        v = __fadd_rn(v, __ldcs(rp)); rp += S1;\n";
            o << "        __stcs(op, v); op += S1; }  // row " << sg.r0 + q << "\n";
        }
        }
        o << "    }\n  }\n}\n";
    }
    o << "extern \"C\" __global__ void __launch_bounds__(W * 32, 1)"
         " spcv_jit(const float* __restrict__ act, float* __restrict__ out,"
         " const float* __restrict__ bias, long long N, long long S, float lo, float hi,"
         " const float* __restrict__ res, u64 one) {\n"
      << "  extern __shared__ float4 smem4[];\n"
      << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
      << "  float* ring = reinterpret_cast<float*>(smem4) + warp * (P * KC * " << 32 * key.cpl << ");\n"
      << "  const int seg = seg_of[blockIdx.x], rank = rank_of[blockIdx.x];\n"
      << "  switch (seg) {\n";
    for (size_t si = 0; si < segs.size(); ++si)
        o << "    case " << si << ": seg" << si << "(act, out, bias, N, S, lo, hi, res, one, ring, lane, "
          << "(long long)rank * W + warp, " << segs[si].ctas * key.warps << "LL); break;\n";
    o << "  }\n}\n";
    return o.str();
}

// Direct variant for small K (<= kJitDirectMaxK): one thread per virtual
// column, 128-thread CTAs, no shared memory and no layout requirement. The
// thread loads its column's activations straight into registers (coalesced
// across the warp), then every row is straight-line code with the weights as
// immediates, 4 rows interleaved term by term; per row the order is the
// reference's (bias first, blocks ascending).
long long direct_instr(int M, int K, int BH, const uint32_t* row_ptr, const JitKey& key) {
    long long weights = 0;
    const int rows = std::min(M, key.m_out);
    for (int r = 0; r < rows; ++r) weights += row_nnz(row_ptr, BH, r);
    return (key.strict ? 2 : 1) * weights + K + 6LL * rows + (key.dw ? 30LL * K : 0);
}

std::string gen_direct(int M, int K, int BH, const uint32_t* row_ptr, const uint32_t* col_idx,
                       const float* values, const JitKey& key) {
    std::ostringstream o;
    auto imm = [](float v) {
        uint32_t u;
        std::memcpy(&u, &v, 4);
        char wv[40];
        std::snprintf(wv, sizeof wv, "__uint_as_float(0x%08xu)", u);
        return std::string(wv);
    };
    o << "extern \"C\" __global__ void __launch_bounds__(128) spcv_jit(const float* __restrict__ act,"
         " float* __restrict__ out, const float* __restrict__ bias, long long N, long long S,"
         " float lo, float hi, const float* __restrict__ res, unsigned long long one,"
         " const float* __restrict__ dwin, int H, int W, int OW, int pt, int pl, float dlo, float dhi) {\n"
      << "  const long long n = blockIdx.x * 128LL + threadIdx.x;\n"
      << "  if (n >= N) return;\n"
      << "  const long long b = n / S, s = n - b * S;\n"
      << "  float* o = out + b * " << key.m_out << "LL * S + s;\n";
    if (key.res) o << "  const float* rp = res + b * " << key.m_out << "LL * S + s;\n";
    std::vector<char> used(static_cast<size_t>(K), 0);
    const int brows = M / BH;
    for (uint32_t b = 0; b < row_ptr[brows]; ++b) used[col_idx[b]] = 1;
    if (!key.dw) {
        o << "  const float* a = act + b * " << K << "LL * S + s;\n";
        for (int k = 0; k < K; ++k)
            if (used[k]) o << "  const float x" << k << " = __ldcs(a + " << k << "LL * S);\n";
    } else {
        // x_k = the depthwise output (channel k, this pixel): bias first, taps
        // in (ky, kx) order, out-of-image taps skipped, ternary clamp
        // (depthwise_conv_chw, kernels.cpp:385-422)
        o << "  const int oy = (int)(s / OW), ox = (int)(s - (long long)oy * OW);\n"
          << "  const int iy0 = oy * " << key.dw_stride << " - pt, ix0 = ox * " << key.dw_stride << " - pl;\n"
          << "  const long long HW = (long long)H * W;\n"
          << "  const float* din = dwin + b * " << K << "LL * HW;\n";
        for (int t = 0; t < 9; ++t)
            o << "  const bool v" << t << " = (unsigned)(iy0 + " << t / 3 << ") < (unsigned)H && (unsigned)(ix0 + "
              << t % 3 << ") < (unsigned)W;\n"
              << "  const long long q" << t << " = v" << t << " ? (long long)(iy0 + " << t / 3 << ") * W + (ix0 + "
              << t % 3 << ") : 0;\n";
        for (int k = 0; k < K; ++k) {
            if (!used[k]) continue;
            o << "  float x" << k << " = " << (key.dw_b ? imm(key.dw_b[k]) : std::string("0.0f")) << ";\n"
              << "  { const float* dk = din + " << k << "LL * HW;\n";
            for (int t = 0; t < 9; ++t)
                o << "    if (v" << t << ") x" << k << " = __fadd_rn(x" << k << ", __fmul_rn("
                  << imm(key.dw_w[static_cast<size_t>(k) * 9 + t]) << ", __ldg(dk + q" << t << ")));\n";
            if (key.dw_clamp)
                o << "    x" << k << " = x" << k << " < dlo ? dlo : (x" << k << " > dhi ? dhi : x" << k << ");\n";
            o << "  }\n";
        }
    }
    constexpr int kIL = 4;
    const int rows = std::min(M, key.m_out);
    for (int r0 = 0; r0 < rows; r0 += kIL) {
        const int r1 = std::min(rows, r0 + kIL);
        o << "  {\n";
        int longest = 0;
        for (int r = r0; r < r1; ++r) {
            longest = std::max(longest, row_nnz(row_ptr, BH, r));
            o << "    float a" << r - r0 << " = "
              << (key.bias ? "__ldg(bias + " + std::to_string(r) + ")" : "0.0f") << ";\n";
        }
        for (int t = 0; t < longest; ++t) {
            for (int r = r0; r < r1; ++r) {
                if (t >= row_nnz(row_ptr, BH, r)) continue;
                const uint32_t blk = row_ptr[r / BH] + static_cast<uint32_t>(t);
                const std::string A = "a" + std::to_string(r - r0);
                float v = values[static_cast<size_t>(blk) * BH + r % BH];
                uint32_t u;
                std::memcpy(&u, &v, 4);
                char wv[40];
                std::snprintf(wv, sizeof wv, "__uint_as_float(0x%08xu)", u);
                const std::string x = "x" + std::to_string(col_idx[blk]);
                if (key.strict)
                    o << "    " << A << " = __fadd_rn(" << A << ", __fmul_rn(" << wv << ", " << x << "));\n";
                else
                    o << "    " << A << " = __fmaf_rn(" << wv << ", " << x << ", " << A << ");\n";
            }
        }
        for (int r = r0; r < r1; ++r) {
            const std::string A = "a" + std::to_string(r - r0);
            if (key.clamp)
                o << "    " << A << " = " << A << " < lo ? lo : (" << A << " > hi ? hi : " << A << ");\n";
            if (key.res) o << "    " << A << " = __fadd_rn(" << A << ", __ldcs(rp + " << r << "LL * S));\n";
            o << "    __stcs(o + " << r << "LL * S, " << A << ");  // row " << r << "\n";
        }
        o << "  }\n";
    }
    o << "}\n";
    return o.str();
}

// Which generator serves (matrix, key): direct for small K within the code
// budget, else the k-major segmented kernel when the layout allows it.
enum class JitKind { kNone, kDirect, kKMajor };
JitKind choose_kind(int M, int K, int BH, const uint32_t* row_ptr, JitKey& key, const Knobs& kn,
                    std::vector<Segment>& segs) {
    // fast mode (1 FFMA per weight) affords the direct variant up to K = 128
    // (measured: MBv1 pw3 in the full step 2.387 -> 2.326 ms); strict keeps
    // K <= 64 there (k-major is faster for pw3 strict)
    const int direct_maxk = knob(kn.jit_direct_maxk, key.strict ? kJitDirectMaxK : 2 * kJitDirectMaxK);
    if (K <= direct_maxk && direct_instr(M, K, BH, row_ptr, key) <= knob(kn.jit_seg_instr, kJitSegInstr))
        return JitKind::kDirect;
    if (!key.vec || key.dw) return JitKind::kNone;
    // k-major: 2 columns per lane (f32x2), or 1 column per lane (scalar, twice
    // the rows per segment) when that fits the matrix in a single segment:
    // every extra segment re-reads the activations (measured, MBv1 pw3 in the
    // full step: 240 -> 199 us; two 1-column segments lose to the tile kernel)
    JitKey k2 = key, k1 = key;
    k2.cpl = 2;
    k1.cpl = 1;
    std::vector<Segment> s2, s1;
    const bool ok2 = plan_segments(M, K, BH, row_ptr, k2, kn, s2);
    const bool ok1 = plan_segments(M, K, BH, row_ptr, k1, kn, s1);
    if (ok1 && s1.size() == 1 && (!ok2 || s2.size() > 1)) {
        segs = s1;  // a single segment reads the activations once
        key.cpl = 1;
        return JitKind::kKMajor;
    }
    if (ok2) {
        segs = s2;
        key.cpl = 2;
        return JitKind::kKMajor;
    }
    return JitKind::kNone;
}

std::mutex g_jit_mu;

// On-disk cubin cache: NVRTC output keyed by a 128-bit hash of the generated
// source (which spells out the matrix, the call shape and the geometry), the
// compile options and the NVRTC version, so a serving process never compiles
// a (matrix, shape) it has compiled before. $SPCV_JIT_CACHE_DIR, else
// $XDG_CACHE_HOME/spcv_b200/jit, else ~/.cache/spcv_b200/jit; SPCV_JIT_CACHE=0
// disables it. Writes are atomic (temporary file + rename); a file that does
// not load is ignored and replaced.
std::string cache_dir() {
    static const std::string dir = [] {
        const char* off = std::getenv("SPCV_JIT_CACHE");
        if (off && std::atoi(off) == 0) return std::string();
        if (const char* d = std::getenv("SPCV_JIT_CACHE_DIR")) return std::string(d);
        if (const char* x = std::getenv("XDG_CACHE_HOME")) return std::string(x) + "/spcv_b200/jit";
        if (const char* h = std::getenv("HOME")) return std::string(h) + "/.cache/spcv_b200/jit";
        return std::string();
    }();
    return dir;
}

std::string cache_name(const std::string& src, const std::vector<const char*>& opts) {
    uint64_t a = 0xcbf29ce484222325ull, b = 0x84222325cbf29ce4ull;  // FNV-1a / a second multiplier
    auto mix = [&](const char* p, size_t n) {
        for (size_t i = 0; i < n; ++i) {
            a = (a ^ static_cast<unsigned char>(p[i])) * 0x100000001b3ull;
            b = (b ^ static_cast<unsigned char>(p[i])) * 0x9E3779B97F4A7C15ull;
            b ^= b >> 29;
        }
    };
    int major = 0, minor = 0;
    nvrtcVersion(&major, &minor);
    const std::string ver = std::to_string(major) + "." + std::to_string(minor);
    mix(ver.data(), ver.size());
    for (const char* o : opts) mix(o, std::strlen(o) + 1);
    mix(src.data(), src.size());
    char buf[64];
    std::snprintf(buf, sizeof buf, "%016llx%016llx.cubin", static_cast<unsigned long long>(a),
                  static_cast<unsigned long long>(b));
    return buf;
}

bool cache_read(const std::string& path, std::vector<char>& out) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    bool ok = n > 0;
    if (ok) {
        out.resize(static_cast<size_t>(n));
        ok = std::fread(out.data(), 1, out.size(), f) == out.size();
    }
    std::fclose(f);
    return ok;
}

void cache_write(const std::string& dir, const std::string& name, const std::vector<char>& cubin) {
    std::string acc;  // mkdir -p
    for (size_t i = 0; i <= dir.size(); ++i) {
        if (i == dir.size() || dir[i] == '/') {
            if (!acc.empty()) mkdir(acc.c_str(), 0755);
        }
        if (i < dir.size()) acc += dir[i];
    }
    const std::string tmp = dir + "/." + name + "." + std::to_string(getpid());
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) return;
    const bool ok = std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
    std::fclose(f);
    if (!ok || std::rename(tmp.c_str(), (dir + "/" + name).c_str()) != 0) std::remove(tmp.c_str());
}

std::vector<const char*> nvrtc_options() {
    static const std::string maxrreg = [] {
        const char* e = std::getenv("SPCV_JIT_MAXRREG");  // tuning knob (occupancy experiments)
        return e ? std::string("--maxrregcount=") + e : std::string();
    }();
    std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=false"};
    if (!maxrreg.empty()) opts.push_back(maxrreg.c_str());
    return opts;
}

}  // namespace

namespace spcv_detail {

std::atomic<uint64_t> g_jit_compiles{0}, g_jit_cache_hits{0};

// NVRTC: source -> sm_100a cubin. No device needed.
int jit_compile(const std::string& src, std::vector<char>& cubin) {
    const std::vector<const char*> opts = nvrtc_options();
    const std::string dir = cache_dir();
    const std::string name = dir.empty() ? std::string() : cache_name(src, opts);
    if (!dir.empty() && cache_read(dir + "/" + name, cubin)) {
        g_jit_cache_hits.fetch_add(1, std::memory_order_relaxed);
        return SPCV_OK;
    }
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "spcv_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
        return fail(SPCV_ERR_UNSUPPORTED, "jit: nvrtcCreateProgram failed");
    if (nvrtcCompileProgram(prog, static_cast<int>(opts.size()), opts.data()) != NVRTC_SUCCESS) {
        size_t n = 0;
        nvrtcGetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        nvrtcGetProgramLog(prog, log.data());
        nvrtcDestroyProgram(&prog);
        return fail(SPCV_ERR_UNSUPPORTED, "jit: compile failed: " + log.substr(0, 400));
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    cubin.resize(n);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    g_jit_compiles.fetch_add(1, std::memory_order_relaxed);
    if (!dir.empty()) cache_write(dir, name, cubin);
    return SPCV_OK;
}

const JitVariant* jit_plan(const spcv_cu_weights* w, const JitKey& key) {
    if (!w || !w->jit_eligible) return nullptr;
    std::lock_guard<std::mutex> lk(g_jit_mu);
    for (const JitVariant& v : w->jit)
        if (v.key == key) return v.eligible ? &v : nullptr;
    w->jit.emplace_back();
    JitVariant& v = w->jit.back();
    v.key = key;
    std::vector<Segment> segs;
    JitKey gk = key;  // plus the generator's choices (columns per lane)
    const JitKind kind = choose_kind(w->rows, w->cols, w->block_h, w->h_row_ptr.data(), gk, w->knobs, segs);
    if (kind == JitKind::kNone) return nullptr;  // the tile kernel runs
    v.eligible = true;
    v.direct = kind == JitKind::kDirect;
    v.cpl = gk.cpl;
    v.segments = static_cast<int>(segs.size());
    return &v;
}

const JitVariant* jit_build(const spcv_cu_weights* w, const JitVariant* cv) {
    if (!cv) return nullptr;
    std::lock_guard<std::mutex> lk(g_jit_mu);
    // the variant lives in w->jit (mutable cache): find the non-const element
    JitVariant* vp = nullptr;
    for (JitVariant& x : w->jit)
        if (&x == cv) vp = &x;
    if (!vp) return nullptr;
    JitVariant& v = *vp;
    if (v.built) return v.fn ? &v : nullptr;
    v.built = true;
    std::vector<Segment> segs;
    JitKey gk = v.key;
    choose_kind(w->rows, w->cols, w->block_h, w->h_row_ptr.data(), gk, w->knobs, segs);  // same plan
    std::vector<char> cubin;
    const std::string src =
        v.direct ? gen_direct(w->rows, w->cols, w->block_h, w->h_row_ptr.data(), w->h_col_idx.data(),
                              w->h_values.data(), v.key)
                 : gen_source(w->rows, w->cols, w->block_h, w->h_row_ptr.data(), w->h_col_idx.data(),
                              w->h_values.data(), gk, w->knobs, segs);
    if (jit_compile(src, cubin) != SPCV_OK) return nullptr;
    cudaError_t e = cudaLibraryLoadData(&v.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e != cudaSuccess) {
        cuda_fail(e, "jit: cudaLibraryLoadData");
        v.lib = nullptr;
        return nullptr;
    }
    e = cudaLibraryGetKernel(&v.fn, v.lib, "spcv_jit");
    if (e == cudaSuccess && !v.direct)
        e = cudaFuncSetAttribute(reinterpret_cast<const void*>(v.fn),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 jit_smem_bytes(v.key.warps, v.key.stages, v.cpl));
    if (e != cudaSuccess) {
        cuda_fail(e, "jit: kernel setup");
        cudaLibraryUnload(v.lib);
        v.lib = nullptr;
        v.fn = nullptr;
        return nullptr;
    }
    return &v;
}

void jit_geometry(JitKey& key, const Knobs& kn) {
    key.warps = knob(kn.jit_warps, kJitWarps);
    key.stages = knob(kn.jit_stages, kJitStages);
    if (key.warps < 1 || key.warps > 32) key.warps = kJitWarps;
    if (key.stages < 1 || key.stages > 8) key.stages = kJitStages;
    while (key.stages > 1 && jit_smem_bytes(key.warps, key.stages) > 227 * 1024) --key.stages;
    while (jit_smem_bytes(key.warps, key.stages) > 227 * 1024) --key.warps;
}

void jit_release(spcv_cu_weights* w) {
    for (JitVariant& v : w->jit)
        if (v.lib) cudaLibraryUnload(v.lib);
    w->jit.clear();
}

int jit_launch(const JitVariant* v, const spcvk::KernelArgs& a, cudaStream_t st, const JitDwArgs* dw) {
    long long N = a.N, S = a.S;
    float lo = a.lo, hi = a.hi;
    const float* act = a.act;
    float* out = a.out;
    const float* bias = a.bias;
    const float* res = a.residual;
    unsigned long long one = 0x3f8000003f800000ULL;  // {1.0f, 1.0f}
    JitDwArgs d = dw ? *dw : JitDwArgs{};
    void* args[] = {&act, &out, &bias, &N, &S, &lo, &hi, &res, &one,
                    &d.in, &d.H, &d.W, &d.OW, &d.pad_t, &d.pad_l, &d.lo, &d.hi};
    cudaLaunchConfig_t cfg = {};
    cfg.stream = st;
    if (v->direct) {
        const long long blocks = (N + 127) / 128;
        if (blocks > 0x7FFFFFFFLL) return fail(SPCV_ERR_UNSUPPORTED, "jit: grid too large");
        cfg.gridDim = dim3(static_cast<unsigned>(blocks));
        cfg.blockDim = dim3(128);
        SPCV_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(v->fn), args));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return SPCV_OK;
    }
    cfg.gridDim = dim3(v->key.sms);
    cfg.blockDim = dim3(v->key.warps * 32);
    cfg.dynamicSmemBytes = jit_smem_bytes(v->key.warps, v->key.stages, v->cpl);
    SPCV_CUDA(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(v->fn), args));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return SPCV_OK;
}

}  // namespace spcv_detail

// Test hook (not in the public header): plan, generate and compile the
// specialised kernel for a host BCSR matrix without a device. Reports the
// number of row segments, source and cubin sizes, and copies up to src_cap
// bytes of source when src_out is non-null (segments = 0: direct variant).
// Returns SPCV_ERR_UNSUPPORTED when the matrix is not eligible.
extern "C" int spcvx_jit_compile(int rows, int cols, int block_h, const uint32_t* row_ptr,
                                 const uint32_t* col_idx, size_t nblocks, const float* values,
                                 int mode, int act_kind, int has_bias, int has_res, int m_out,
                                 int sms, int* segments, size_t* src_bytes, size_t* cubin_bytes,
                                 char* src_out, size_t src_cap) {
    (void)nblocks;
    JitKey key;
    key.strict = mode == SPCV_MODE_STRICT;
    key.clamp = act_kind == SPCV_ACT_CLAMP;
    key.bias = has_bias != 0;
    key.res = has_res != 0;
    key.m_out = m_out;
    key.vec = true;
    key.sms = sms;
    const Knobs kn = Knobs::from_env();
    spcv_detail::jit_geometry(key, kn);
    std::vector<Segment> segs;
    const JitKind kind = choose_kind(rows, cols, block_h, row_ptr, key, kn, segs);
    if (kind == JitKind::kNone) return SPCV_ERR_UNSUPPORTED;
    if (segments) *segments = kind == JitKind::kDirect ? 0 : static_cast<int>(segs.size());
    const std::string src = kind == JitKind::kDirect
                                ? gen_direct(rows, cols, block_h, row_ptr, col_idx, values, key)
                                : gen_source(rows, cols, block_h, row_ptr, col_idx, values, key, kn, segs);
    if (src_bytes) *src_bytes = src.size();
    if (src_out && src_cap) {
        const size_t n = std::min(src_cap - 1, src.size());
        std::memcpy(src_out, src.data(), n);
        src_out[n] = '\0';
    }
    std::vector<char> cubin;
    const int rc = spcv_detail::jit_compile(src, cubin);
    if (cubin_bytes) *cubin_bytes = cubin.size();
    return rc;
}
