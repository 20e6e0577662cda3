/*
 * spcv_oracle.c — CPU restatement of the reference SpMM path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_1911_09723_b200/,
 * include/) links, imports or calls this file. Only tests/, the smoke() check in
 * __graft_entry__.py and bench.py's cpu_baseline / --impl reference legs use it,
 * and only as the checker or the reported CPU baseline.
 *
 * Pinned against: the reference itself compiled from /root/reference by
 * oracle/Makefile into oracle/_ref/ (tests/test_oracle.py compares the two
 * bit-for-bit), and the golden fixtures in tests/golden/ generated from the
 * reference by tests/golden/make_golden.py.
 *
 * Build flags matter: -O2 -ffp-contract=off, no -march=native. With FMA
 * contraction the reference itself stops being bit-exact against its own
 * dense oracle.
 *
 * Every function cites the reference lines it restates.
 */
#include <math.h>
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Error codes shared with include/spcv_cu.h (SPCV_OK ... SPCV_ERR_INVALID). */
enum {
    OR_OK = 0,
    OR_ERR_LAYOUT = 1,
    OR_ERR_SHAPE = 2,
    OR_ERR_FORMAT = 3,
    OR_ERR_INVALID = 4,
};

/* Activation kinds: 0 = None, 1 = Clamp(lo, hi). */

/* Activation::apply — /root/reference/proj/include/spcv/tensor.hpp:90-96.
 * Ternary compare: NaN passes through, -0.0 is preserved. */
static inline float or_apply(int kind, float lo, float hi, float x) {
    if (kind == 1) {
        if (x < lo) return lo;
        if (x > hi) return hi;
    }
    return x;
}

/* matmul_reference — /root/reference/proj/src/tensor.cpp:38-62.
 * out[c][s] = act(bias[c] + sum_k w[c][k] * in[k][s]), bias first, k
 * ascending, separate multiply and add, every (including zero) weight visited.
 * w is rows x cols row-major; act is [cols][S]; out is [rows][S]. */
int oracle_matmul_reference(int rows, int cols, int S, const float* w, const float* act,
                            const float* bias, int act_kind, float lo, float hi, float* out) {
    if (rows < 0 || cols < 1 || S < 1) return OR_ERR_SHAPE;
    for (int c = 0; c < rows; ++c) {
        float* dst = out + (size_t)c * S;
        const float b = bias ? bias[c] : 0.0f;
        for (int s = 0; s < S; ++s) dst[s] = b;
        for (int k = 0; k < cols; ++k) {
            const float wv = w[(size_t)c * cols + k];
            const float* src = act + (size_t)k * S;
            for (int s = 0; s < S; ++s) {
                const float p = wv * src[s];
                dst[s] = dst[s] + p;
            }
        }
        if (act_kind != 0)
            for (int s = 0; s < S; ++s) dst[s] = or_apply(act_kind, lo, hi, dst[s]);
    }
    return OR_OK;
}

/* Per-element semantics of spmm_into's strip microkernels —
 * /root/reference/proj/src/kernels.cpp:14-43 (scalar) and 101-130 (vector):
 * acc = bias (or +0.0 when bias is null, kernels.cpp:21,110); for each stored
 * block of the block row in ascending position, acc += value * act[col][s]
 * (mul then add, kernels.cpp:30,120); then the ternary clamp
 * (kernels.cpp:38, 93-99). Strip width and tier never change the per-element
 * order, so one scalar loop restates every variant. */
int oracle_spmm_bcsr(int rows, int cols, int block_h, const uint32_t* row_ptr,
                     const uint32_t* col_idx, const float* values, int S, const float* act,
                     const float* bias, int act_kind, float lo, float hi, float* out) {
    if (block_h != 1 && block_h != 2 && block_h != 4) return OR_ERR_FORMAT;
    if (rows % block_h != 0) return OR_ERR_FORMAT;
    (void)cols;
    const int brows = rows / block_h;
    for (int br = 0; br < brows; ++br) {
        for (int n = 0; n < block_h; ++n) {
            const int r = br * block_h + n;
            float* dst = out + (size_t)r * S;
            const float b = bias ? bias[r] : 0.0f;
            for (int s = 0; s < S; ++s) dst[s] = b;
            for (uint32_t blk = row_ptr[br]; blk < row_ptr[br + 1]; ++blk) {
                const float wv = values[(size_t)blk * block_h + n];
                const float* src = act + (size_t)col_idx[blk] * S;
                for (int s = 0; s < S; ++s) {
                    const float p = wv * src[s];
                    dst[s] = dst[s] + p;
                }
            }
            for (int s = 0; s < S; ++s) dst[s] = or_apply(act_kind, lo, hi, dst[s]);
        }
    }
    return OR_OK;
}

/* Batch of independent images: act [images][cols][S], out [images][rows][S].
 * The reference is single-image (tensor.hpp:28-29); a batch is a loop of
 * per-image calls. Images [i0, i1) only. */
static void spmm_images(int rows, int cols, int block_h, const uint32_t* row_ptr,
                        const uint32_t* col_idx, const float* values, int i0, int i1, int S,
                        const float* act, const float* bias, int act_kind, float lo, float hi,
                        float* out) {
    for (int i = i0; i < i1; ++i)
        oracle_spmm_bcsr(rows, cols, block_h, row_ptr, col_idx, values, S,
                         act + (size_t)i * cols * S, bias, act_kind, lo, hi,
                         out + (size_t)i * rows * S);
}

typedef struct {
    int rows, cols, block_h, i0, i1, S, act_kind;
    const uint32_t *row_ptr, *col_idx;
    const float *values, *act, *bias;
    float lo, hi;
    float* out;
} or_job;

static void* or_worker(void* p) {
    const or_job* j = (const or_job*)p;
    spmm_images(j->rows, j->cols, j->block_h, j->row_ptr, j->col_idx, j->values, j->i0, j->i1,
                j->S, j->act, j->bias, j->act_kind, j->lo, j->hi, j->out);
    return NULL;
}

/* Images partitioned contiguously over nthreads host threads (reentrancy per
 * /root/reference/SPEC.md:290). Used as the "port" CPU baseline when the
 * compiled reference is unavailable. */
int oracle_spmm_bcsr_batched(int rows, int cols, int block_h, const uint32_t* row_ptr,
                             const uint32_t* col_idx, const float* values, int images, int S,
                             const float* act, const float* bias, int act_kind, float lo,
                             float hi, float* out, int nthreads) {
    if (block_h != 1 && block_h != 2 && block_h != 4) return OR_ERR_FORMAT;
    if (rows % block_h != 0) return OR_ERR_FORMAT;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > images) nthreads = images > 0 ? images : 1;
    if (nthreads == 1) {
        spmm_images(rows, cols, block_h, row_ptr, col_idx, values, 0, images, S, act, bias,
                    act_kind, lo, hi, out);
        return OR_OK;
    }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    or_job* jobs = (or_job*)malloc(sizeof(or_job) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        or_job j = {rows, cols, block_h, (int)((long)images * t / nthreads),
                    (int)((long)images * (t + 1) / nthreads), S, act_kind, row_ptr, col_idx,
                    values, act, bias, lo, hi, out};
        jobs[t] = j;
        pthread_create(&th[t], NULL, or_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return OR_OK;
}

/* encode_bcsr — /root/reference/proj/src/sparse.cpp:108-134. A block is kept
 * iff any of its block_h members is nonzero (!= 0.0f, so -0.0 counts as zero);
 * kept blocks store all members (explicit zeros inside blocks), values are
 * block-contiguous, output-channel-minor. Caller sizes col_idx for rows/bh*cols
 * blocks and values for rows*cols entries; *nblocks receives the block count. */
int oracle_encode_bcsr(int rows, int cols, int block_h, const float* w, uint32_t* row_ptr,
                       uint32_t* col_idx, float* values, size_t* nblocks) {
    if (block_h != 1 && block_h != 2 && block_h != 4) return OR_ERR_FORMAT;
    if (rows % block_h != 0) return OR_ERR_SHAPE;
    const int brows = rows / block_h;
    size_t nb = 0;
    row_ptr[0] = 0;
    for (int br = 0; br < brows; ++br) {
        for (int c = 0; c < cols; ++c) {
            int keep = 0;
            for (int n = 0; n < block_h && !keep; ++n)
                if (w[(size_t)(br * block_h + n) * cols + c] != 0.0f) keep = 1;
            if (!keep) continue;
            col_idx[nb] = (uint32_t)c;
            for (int n = 0; n < block_h; ++n)
                values[nb * block_h + n] = w[(size_t)(br * block_h + n) * cols + c];
            ++nb;
        }
        row_ptr[br + 1] = (uint32_t)nb;
    }
    *nblocks = nb;
    return OR_OK;
}

/* BcsrMatrix::validate — /root/reference/proj/src/sparse.cpp:16-51, same
 * checks in the same order; every failure is a FormatError. */
int oracle_validate_bcsr(int rows, int cols, int block_h, const uint32_t* row_ptr,
                         size_t row_ptr_len, const uint32_t* col_idx, size_t nblocks,
                         size_t nvalues) {
    if (rows < 1 || cols < 1) return OR_ERR_FORMAT;
    if (block_h != 1 && block_h != 2 && block_h != 4) return OR_ERR_FORMAT;
    if (rows % block_h != 0) return OR_ERR_FORMAT;
    const size_t brows = (size_t)(rows / block_h);
    if (row_ptr_len != brows + 1) return OR_ERR_FORMAT;
    if (row_ptr[0] != 0) return OR_ERR_FORMAT;
    for (size_t r = 0; r < brows; ++r)
        if (row_ptr[r] > row_ptr[r + 1]) return OR_ERR_FORMAT;
    if (row_ptr[brows] != nblocks) return OR_ERR_FORMAT;
    if (nvalues != nblocks * (size_t)block_h) return OR_ERR_FORMAT;
    for (size_t r = 0; r < brows; ++r) {
        uint32_t prev = 0;
        int first = 1;
        for (uint32_t b = row_ptr[r]; b < row_ptr[r + 1]; ++b) {
            const uint32_t c = col_idx[b];
            if (c >= (uint32_t)cols) return OR_ERR_FORMAT;
            if (!first && c <= prev) return OR_ERR_FORMAT;
            prev = c;
            first = 0;
        }
    }
    return OR_OK;
}

/* decode_bcsr — /root/reference/proj/src/sparse.cpp:136-148: validate, then
 * scatter the stored blocks into a zeroed rows x cols matrix. */
int oracle_decode_bcsr(int rows, int cols, int block_h, const uint32_t* row_ptr,
                       size_t row_ptr_len, const uint32_t* col_idx, size_t nblocks,
                       const float* values, size_t nvalues, float* w) {
    const int rc = oracle_validate_bcsr(rows, cols, block_h, row_ptr, row_ptr_len, col_idx,
                                        nblocks, nvalues);
    if (rc != OR_OK) return rc;
    memset(w, 0, sizeof(float) * (size_t)rows * cols);
    const int brows = rows / block_h;
    for (int br = 0; br < brows; ++br)
        for (uint32_t b = row_ptr[br]; b < row_ptr[br + 1]; ++b)
            for (int n = 0; n < block_h; ++n)
                w[(size_t)(br * block_h + n) * cols + col_idx[b]] = values[(size_t)b * block_h + n];
    return OR_OK;
}
