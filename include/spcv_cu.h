/*
 * spcv_cu.h — C-ABI boundary of the B200 sparse 1x1-conv SpMM.
 *
 * This is the drop-in for the reference's hot path
 *   spcv::spmm_into / spcv::spmm / spcv::spconv_1x1
 *   (/root/reference/proj/include/spcv/kernels.hpp:45-55,
 *    implementation /root/reference/proj/src/kernels.cpp:304-341)
 * consuming the reference's BCSR weight format
 *   spcv::BcsrMatrix (/root/reference/proj/include/spcv/sparse.hpp:65-79).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary and
 * no exception escapes it. Every entry point returns an spcv_status; the
 * message for the last failure on the calling thread is spcv_cu_last_error().
 * The C++ mirror of the reference API (include/spcv_b200/spcv.hpp) maps the
 * codes back onto the reference's exception classes.
 *
 * Arithmetic contract: SPCV_MODE_STRICT reproduces the reference per-element
 * order (bias first, stored blocks in ascending position, separate multiply
 * and add, ternary clamp) and is bit-exact against the reference CPU kernel.
 * SPCV_MODE_FAST contracts multiply+add into FFMA and is within the
 * nnz-scaled 1e-5 tolerance of BASELINE.json's north_star.
 */
#ifndef SPCV_CU_H
#define SPCV_CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The numbering is shared with the CPU checkers in oracle/. */
typedef enum spcv_status {
    SPCV_OK = 0,
    SPCV_ERR_LAYOUT = 1,   /* spcv::LayoutError      (tensor.hpp:18-21)   */
    SPCV_ERR_SHAPE = 2,    /* spcv::ShapeError       (tensor.hpp:12-15)   */
    SPCV_ERR_FORMAT = 3,   /* spcv::FormatError      (sparse.hpp:12-15)   */
    SPCV_ERR_INVALID = 4,  /* std::invalid_argument  (kernels.cpp:321-322) */
    SPCV_ERR_CUDA = 5,     /* CUDA runtime failure (no device, launch error, ...) */
    SPCV_ERR_UNSUPPORTED = 6, /* shape beyond this build's device limits */
    /* model files (model_io.hpp:13-46) */
    SPCV_ERR_MODEL_IO = 7,     /* spcv::ModelIoError (generic)                 */
    SPCV_ERR_BAD_MAGIC = 8,    /* spcv::BadMagicError                          */
    SPCV_ERR_VERSION = 9,      /* spcv::UnsupportedVersionError                */
    SPCV_ERR_TRUNCATED = 10,   /* spcv::TruncatedError                         */
    SPCV_ERR_CHECKSUM = 11,    /* spcv::ChecksumError                          */
    SPCV_ERR_MODEL_FORMAT = 12 /* spcv::ModelFormatError                       */
} spcv_status;

/* Tensor layouts, as spcv::Layout (tensor.hpp:23-26). */
enum { SPCV_LAYOUT_CHW = 0, SPCV_LAYOUT_HWC = 1 };

/* Fused activation kinds, as spcv::Activation::Kind (tensor.hpp:74-97).
 * SPCV_ACT_CLAMP requires lo < hi (tensor.hpp:80-81). ReLU = clamp(0, +inf),
 * ReLU6 = clamp(0, 6). */
enum { SPCV_ACT_NONE = 0, SPCV_ACT_CLAMP = 1 };

/* Arithmetic modes. */
enum { SPCV_MODE_STRICT = 0, SPCV_MODE_FAST = 1 };

/* Opaque device-resident packed weights (one BcsrMatrix, one device). */
typedef struct spcv_cu_weights spcv_cu_weights;

/* Pack a reference BcsrMatrix (host arrays, exactly the fields of
 * sparse.hpp:65-79) into device-resident streams on the current CUDA device:
 * per-block-row nnz counts, per-block input-channel deltas and the block
 * values (the paper's format), plus the row-bucketed execution schedule.
 * The matrix is validated with the checks of BcsrMatrix::validate
 * (sparse.cpp:16-51); a malformed matrix yields SPCV_ERR_FORMAT.
 * Replaces: the per-call use of `const BcsrMatrix& w` in spmm_into
 * (kernels.cpp:304). */
int spcv_cu_pack(int rows, int cols, int block_h, const uint32_t* row_ptr, size_t row_ptr_len,
                 const uint32_t* col_idx, size_t nblocks, const float* values, size_t nvalues,
                 spcv_cu_weights** out);

/* Decode the device streams back into BCSR host arrays (row_ptr has
 * rows/block_h+1 entries, col_idx nblocks, values nblocks*block_h). The
 * decode runs on the device and is bit-exact: pack followed by unpack
 * reproduces the input arrays byte for byte. */
int spcv_cu_unpack(const spcv_cu_weights* w, uint32_t* row_ptr, uint32_t* col_idx,
                   float* values);

/* Shape of packed weights; any out-pointer may be NULL. */
int spcv_cu_weights_info(const spcv_cu_weights* w, int* rows, int* cols, int* block_h,
                         size_t* nblocks, int* row_slots, int* device);

void spcv_cu_free(spcv_cu_weights* w);

/* Which CUDA kernel spmm runs for these weights in `mode`:
 *   SPCV_KERNEL_TILE — the shared-memory tile kernel (any K: wide matrices run
 *                      as channel passes that continue each other's sums);
 *   SPCV_KERNEL_JIT  — a kernel specialised on this matrix's structure and
 *                      values (weights as instruction immediates), compiled
 *                      with NVRTC on first use and cached in the weights:
 *                      one thread per column for K <= 64, else k-major row
 *                      segments (S % 4 == 0 layouts) while the code fits the
 *                      instruction-cache budget (jit.cu).
 * Compiles the specialised kernel if it is due and not built yet (probing the
 * spmm_into call shape). Both kernels are bit-exact in SPCV_MODE_STRICT.
 * SPCV_JIT=0 in the environment at pack time selects the tile kernel. No
 * reference counterpart (introspection). */
enum { SPCV_KERNEL_TILE = 0, SPCV_KERNEL_JIT = 1, SPCV_KERNEL_SMALL = 2 };
int spcv_cu_weights_kernel(spcv_cu_weights* w, int mode, int* kernel);

/* The kernel a spmm_into call of `images` act_h x act_w images (16 B-aligned
 * tensors, bias, clamp) runs, which also depends on the column count:
 *   SPCV_KERNEL_JIT     — as above (the k-major variant only with enough
 *                         column groups for its persistent CTAs);
 *   SPCV_KERNEL_SMALL   — fewer column tiles than SMs and <= 8 M products
 *                         (batch 1, small planes): one warp per block row x
 *                         32 columns, activations gathered from global
 *                         memory, no staging (small.cu);
 *   SPCV_KERNEL_TILE    — everything else.
 * All are bit-exact in SPCV_MODE_STRICT. SPCV_SMALL=0|2 at pack time
 * disables / forces the few-column kernel. Compiles the JIT
 * kernel if it is due. No reference counterpart (introspection). */
int spcv_cu_weights_kernel_for(spcv_cu_weights* w, int mode, int images, int act_h, int act_w, int* kernel);

/* spmm_into over a batch of `images` CHW images on device memory:
 *   act [images][act_c][act_h*act_w], out [images][out_c][out_h*out_w].
 *   out[i][c][s] = fused(bias[c] + sum over c's stored blocks of value*act[i][col][s])
 * Checks, in the reference order (kernels.cpp:306-322): clamp lo<hi
 * (tensor.hpp:80-81) -> act layout CHW (LayoutError) -> w.cols == act_c
 * (ShapeError) -> cfg_n == block_h (FormatError) -> bias_len == 0 or rows
 * (ShapeError) -> out CHW with out_c == rows and out spatial == act spatial
 * (ShapeError) -> cfg_m in {0,4,8,16} (invalid_argument). cfg_m is the CPU
 * strip width; it is validated and otherwise ignored (one CUDA path). bias may
 * be NULL (bias_len 0) meaning +0.0 (kernels.cpp:21,110). Asynchronous on
 * `stream` (a cudaStream_t, NULL = legacy default stream). */
int spcv_cu_spmm_into(const spcv_cu_weights* w, const float* act, int act_layout, int images,
                      int act_c, int act_h, int act_w, const float* bias, size_t bias_len,
                      int act_kind, float lo, float hi, float* out, int out_layout, int out_c,
                      int out_h, int out_w, int cfg_m, int cfg_n, int mode, void* stream);

/* Same contract with HOST act/bias/out buffers: host->device copy, kernel,
 * device->host copy, synchronous. This is the reference-facing call shape
 * (spmm_into with host Tensors). Pinned host buffers give full PCIe speed. */
int spcv_cu_spmm_into_host(const spcv_cu_weights* w, const float* act, int act_layout,
                           int images, int act_c, int act_h, int act_w, const float* bias,
                           size_t bias_len, int act_kind, float lo, float hi, float* out,
                           int out_layout, int out_c, int out_h, int out_w, int cfg_m, int cfg_n,
                           int mode);

/* The reference call shape in one call: spmm_into(const BcsrMatrix&, act,
 * bias, fused, out, cfg) (kernels.hpp:45-46) with the matrix as host BCSR
 * arrays (sparse.hpp:65-79) and HOST tensors. Arguments are checked first, in
 * the reference order (as spcv_cu_spmm_into), before the matrix is read; the
 * matrix is then validated (SPCV_ERR_FORMAT) and packed ONCE per distinct
 * content and device: later calls with the same arrays find it in an LRU
 * cache (verified byte for byte; SPCV_WEIGHT_CACHE_MB bounds the cache, 256 by
 * default), so a caller looping spmm_into over layers and images never
 * repacks or recompiles. Replaces: spmm_into (kernels.cpp:304-334) as the
 * reference's callers use it (run_network netdef.cpp:497, bench_layers
 * bench.cpp:209, run_verify bench.cpp:365). */
int spcv_cu_spmm_bcsr_into_host(int rows, int cols, int block_h, const uint32_t* row_ptr,
                                size_t row_ptr_len, const uint32_t* col_idx, size_t nblocks,
                                const float* values, size_t nvalues, const float* act, int act_layout,
                                int images, int act_c, int act_h, int act_w, const float* bias,
                                size_t bias_len, int act_kind, float lo, float hi, float* out,
                                int out_layout, int out_c, int out_h, int out_w, int cfg_m, int cfg_n,
                                int mode);

/* Drop every matrix cached by spcv_cu_spmm_bcsr_into_host. */
void spcv_cu_weight_cache_clear(void);

/* Cache counters (any pointer may be NULL): cached matrices, hits and misses
 * of spcv_cu_spmm_bcsr_into_host, NVRTC compiles of weight-specialised
 * kernels and how many of those were served from the on-disk cubin cache
 * ($SPCV_JIT_CACHE_DIR or ~/.cache/spcv_b200/jit; SPCV_JIT_CACHE=0 disables). */
int spcv_cu_cache_stats(size_t* entries, uint64_t* hits, uint64_t* misses, uint64_t* jit_compiles,
                        uint64_t* jit_disk_hits);

/* The network executor's pointwise step (run_network, netdef.cpp:494-512) on
 * device tensors, fused: weights may carry padded rows (w.rows > out_c, up to
 * block_h-1 extra rows; they are computed with bias 0 and never stored, i.e.
 * the "run wide, keep the logical prefix" of netdef.cpp:496-505), and an
 * optional residual [images][out_c][H*W] is added after the activation
 * (add_residual, netdef.cpp:448-452,512: out = act(acc) + res, separately
 * rounded). bias has out_c entries or none. act [images][act_c][H*W], out
 * [images][out_c][H*W]. Same arithmetic modes as spcv_cu_spmm_into. */
int spcv_cu_spmm_layer(const spcv_cu_weights* w, const float* act, int images, int act_c,
                       int act_h, int act_w, const float* bias, size_t bias_len, int act_kind,
                       float lo, float hi, const float* residual, float* out, int out_c, int mode,
                       void* stream);

/* Dense fp32 baseline with the same contract as the SpMM entry point: the
 * reference's dense_gemm_into (kernels.hpp:85-90, kernels.cpp:345-373), its
 * in-repo speed baseline for the sparse kernel (bench.cpp:216-227). `w` is a
 * DEVICE rows x cols row-major matrix; act/out/bias are device tensors as in
 * spcv_cu_spmm_into. Computed by cuBLAS SGEMM (pedantic fp32, no TF32) plus a
 * fused bias+clamp epilogue kernel: not bit-exact (cuBLAS's summation order),
 * within fp32 rounding of the dense oracle. Checks in the reference order
 * (kernels.cpp:347-360): layout -> cols -> bias -> out shape -> strip width. */
int spcv_cu_dense_gemm_into(const float* w, int rows, int cols, const float* act, int act_layout,
                            int images, int act_c, int act_h, int act_w, const float* bias,
                            size_t bias_len, int act_kind, float lo, float hi, float* out,
                            int out_layout, int out_c, int out_h, int out_w, int cfg_m,
                            void* stream);

/* ---- SPCV model files -------------------------------------
 * The reference's model container ("SPCV" magic, u16 version 1, network
 * descriptor, layer records, CRC-32 trailer; model_io.hpp:48-55) parsed with
 * parse_model's checks in its order (model_io.cpp:238-381) and its typed
 * errors (SPCV_ERR_BAD_MAGIC ... SPCV_ERR_MODEL_FORMAT). */
typedef struct spcv_cu_model spcv_cu_model;

/* Parse and fully validate without touching the device; *layers = count. */
int spcv_cu_model_parse(const uint8_t* bytes, size_t size, int* layers);

/* Parse, then upload once: every sparse 1x1 / classifier layer is packed
 * (spcv_cu_pack) with its bias; dense ones are uploaded row-major. */
int spcv_cu_model_load(const uint8_t* bytes, size_t size, spcv_cu_model** out);

/* Layer i: info[12] = {kind (0 entry, 1 pointwise, 2 depthwise, 3 pool,
 * 4 classifier), cin, cout, in_h, in_w, out_h, out_w, is_sparse, block_h,
 * act_kind, residual_src, stride}. */
int spcv_cu_model_layer(const spcv_cu_model* m, int i, int* info);

/* Borrowed packed weights of sparse layer i (owned by the model). */
int spcv_cu_model_weights(const spcv_cu_model* m, int i, const spcv_cu_weights** w);

/* Run layer i of the executor on device tensors. A 1x1 / classifier layer
 * runs as run_network's pointwise step (netdef.cpp:494-512): its bias, fused
 * activation, padded-row truncation, and the residual (device
 * [images][cout][out_h*out_w], required iff the layer has a residual source).
 * An entry convolution (act: HWC images), depthwise 3x3 (depthwise_conv_chw,
 * kernels.cpp:385-422) or global-pool layer runs as in
 * spcv_cu_model_forward (residual ignored). act [images][cin][in_h*in_w]
 * (CHW) on device; out [images][cout][out_h*out_w]. */
int spcv_cu_model_run(const spcv_cu_model* m, int i, const float* act, int images,
                      const float* residual, float* out, int mode, void* stream);

/* The whole network (run_network, netdef.cpp:456-524) on the device: `images`
 * HWC images input[images][in_h][in_w][in_c] (device memory) -> logits
 * [images][num_classes] (device memory). Every activation stays in HBM; the
 * entry convolution, depthwise 3x3, global pooling, residual adds and the
 * sparse 1x1 / classifier layers (spcv_cu_spmm_layer) run as CUDA kernels, in
 * stream order on `stream`, with a stream-ordered workspace. In
 * SPCV_MODE_STRICT the logits are bit-identical to the reference's
 * run_network; SPCV_MODE_FAST uses fused multiply-adds (SpMM, entry and
 * depthwise convolutions) and cuBLAS for dense 1x1 layers. Serving: a call
 * repeated with the same (images <= 16, input, logits, mode) on the same
 * non-default stream is captured once into a CUDA graph (over a persistent
 * workspace kept until spcv_cu_model_free) and replayed from then on;
 * SPCV_MODEL_GRAPH=0 disables it, a stream that is already capturing gets
 * plain launches. Input dims other than the model's -> SPCV_ERR_SHAPE
 * (check_run_inputs, netdef.cpp:433-441). */
int spcv_cu_model_forward(const spcv_cu_model* m, const float* input, int images, int in_h,
                          int in_w, int in_c, float* logits, int mode, void* stream);

void spcv_cu_model_free(spcv_cu_model* m);

/* Number of SpMM kernel launches issued by this library so far (process-wide). */
uint64_t spcv_cu_launch_count(void);

/* Message describing the last failure on the calling thread ("" if none). */
const char* spcv_cu_last_error(void);

/* Library build string (arch, version). */
const char* spcv_cu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SPCV_CU_H */
