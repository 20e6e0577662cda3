// model_internal.h — the parsed SPCV model (model.cu) as the device
// executor (network.cu) sees it.
#pragma once

#include <cstdint>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "spcv_internal.h"

namespace spcv_model {

enum Kind : uint8_t { kEntryConv = 0, kPointwise = 1, kDepthwise = 2, kGlobalPool = 3, kFullyConnected = 4 };
enum Storage : uint8_t { kNone = 0, kConv = 1, kDw = 2, kDense = 3, kBcsr = 4 };

struct Layer {
    uint8_t kind = 0;
    std::string name;
    int cin = 0, cout = 0, stride = 1, in_h = 0, in_w = 0, out_h = 0, out_w = 0;
    bool sparse = false;
    double sparsity = 0.0;
    int block_h = 1;
    int act_kind = 0;
    float lo = 0.0f, hi = 0.0f;
    int residual_src = -1;
    std::vector<float> bias;
    uint8_t storage = kNone;
    // pointwise / classifier weights
    int rows = 0, cols = 0, bh = 1;
    std::vector<uint32_t> row_ptr, col_idx;
    std::vector<float> values;  // BCSR values or dense row-major data
    // entry conv [co][ci][3][3] / depthwise [c][3][3] weights
    std::vector<float> other;
    // entry / depthwise: finite weights and no -0.0 bias, so out-of-image taps
    // may be read as 0 instead of skipped without changing a bit (network.cu)
    bool zero_pad_exact = false;
};

struct Net {
    std::string name;
    int width_milli = 0, input_h = 0, input_w = 0, input_c = 0, num_classes = 0;
    double plan_sparsity = 0.0;
    int block_start = 0, block_h_after = 0;
    std::vector<Layer> layers;
};

}  // namespace spcv_model

struct spcv_cu_model;
namespace spcv_model {
// network.cu: one entry-convolution, depthwise or global-pool layer on device
// tensors (SPCV_ERR_INVALID for other kinds).
int run_spatial_layer(const spcv_cu_model* m, size_t i, const float* in, int images, float* out, int mode,
                      cudaStream_t st);
}  // namespace spcv_model

struct spcv_cu_model {
    spcv_model::Net net;
    int device = 0;
    std::vector<spcv_cu_weights*> w;  // per layer: packed sparse weights (or null)
    std::vector<float*> d_dense;      // per layer: dense row-major matrix (or null)
    std::vector<float*> d_bias;       // per layer: bias (or null)
    std::vector<float*> d_conv;       // per layer: entry conv [co][ky][kx][ci] / depthwise [c][9]
    // forward() workspace: a stream-ordered pool owned by the model that keeps
    // its memory between calls (no re-mapping per forward)
    cudaMemPool_t pool = nullptr;
    // forward() replayed as a CUDA graph per (images, input, logits, mode,
    // stream) for small batches (network.cu)
    struct GraphKey {
        int images = 0, mode = 0;
        const float* input = nullptr;
        float* logits = nullptr;
        cudaStream_t stream = nullptr;
        bool operator==(const GraphKey& o) const {
            return images == o.images && mode == o.mode && input == o.input && logits == o.logits &&
                   stream == o.stream;
        }
    };
    struct GraphEntry {
        GraphKey key;
        int uses = 0;
        cudaGraphExec_t exec = nullptr;
        cudaEvent_t done = nullptr;  // recorded after the entry's last forward / replay
        bool failed = false;
        uint64_t launches = 0;
        std::vector<float*> ws;  // persistent workspace (model pool) the graph reads and writes
    };
    mutable std::mutex graph_mu;
    mutable std::deque<GraphEntry> graphs;  // least recently used first
    mutable std::deque<GraphKey> seen;      // keys seen once (no entry yet), least recent first
};

