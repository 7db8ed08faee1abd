// synth_kernels.cu — materialise the synthetic model's weights in HBM.
//
// Weights are generated on device straight into their serving layout (one
// pass over HBM, ~TB/s), so loading a 34B-shape prefix takes milliseconds
// instead of a host-side generation plus PCIe copy.
#include "kernels.h"
#include "synth.cuh"

namespace eeb {

namespace {

struct FillArgs {
    uint64_t seed;
    int kind;        // 0 linear, 1 norm gain, 2 embedding, 3 head
    int tid;         // tensor id (linear / norm)
    int rows, cols;  // matrix shape (norm: rows = 1)
    float scale;     // linear scale or head alpha
    int zero_signal_rows;
    int d;
    int exit_index;
    uint32_t vocab, pmul;
    int row0, col0, full_cols;  // slice of a larger tensor (tensor parallelism); full_cols 0 = cols
};

template <typename T>
__global__ void fill_kernel(T* dst, FillArgs a) {
    const int64_t n = (int64_t)a.rows * a.cols;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(idx / a.cols) + a.row0;
        const int c = (int)(idx % a.cols) + a.col0;
        const int fc = a.full_cols > 0 ? a.full_cols : a.cols;
        float v;
        switch (a.kind) {
            case 0:
                v = synth::linear_value(a.seed, a.tid, r, c, fc, a.scale, a.zero_signal_rows != 0, a.d);
                break;
            case 1: v = synth::norm_gain(a.seed, a.tid, c); break;
            case 2: v = synth::emb_value(a.seed, a.d, r, c); break;
            default:
                v = synth::head_value(a.seed, a.d, a.exit_index, a.scale, r, c, a.vocab, a.pmul);
                break;
        }
        dst[idx] = from_f32<T>(v);
    }
}

template <typename T>
void launch_fill(void* dst, const FillArgs& a, cudaStream_t s) {
    const int64_t n = (int64_t)a.rows * a.cols;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    fill_kernel<T><<<(int)blocks, 256, 0, s>>>(static_cast<T*>(dst), a);
    EEB_CHECK_LAUNCH();
}

void fill(int dtype, void* dst, const FillArgs& a, cudaStream_t s) {
    if (dtype == 0) launch_fill<float>(dst, a, s);
    else launch_fill<__nv_bfloat16>(dst, a, s);
}

}  // namespace

void synth_linear(int dtype, void* dst, uint64_t seed, int tid, int rows, int cols, float scale,
                  bool zero_signal_rows, int d, cudaStream_t s) {
    FillArgs a{};
    a.seed = seed; a.kind = 0; a.tid = tid; a.rows = rows; a.cols = cols; a.scale = scale;
    a.zero_signal_rows = zero_signal_rows ? 1 : 0; a.d = d;
    fill(dtype, dst, a, s);
}

void synth_linear_slice(int dtype, void* dst, uint64_t seed, int tid, int rows, int cols, int row0, int col0,
                        int full_cols, float scale, bool zero_signal_rows, int d, cudaStream_t s) {
    FillArgs a{};
    a.seed = seed; a.kind = 0; a.tid = tid; a.rows = rows; a.cols = cols; a.scale = scale;
    a.zero_signal_rows = zero_signal_rows ? 1 : 0; a.d = d;
    a.row0 = row0; a.col0 = col0; a.full_cols = full_cols;
    fill(dtype, dst, a, s);
}

void synth_norm(void* dst_f32, uint64_t seed, int tid, int d, cudaStream_t s) {
    FillArgs a{};
    a.seed = seed; a.kind = 1; a.tid = tid; a.rows = 1; a.cols = d; a.d = d;
    fill(0, dst_f32, a, s);  // norm gains are always f32
}

void synth_embedding(int dtype, void* dst, uint64_t seed, int vocab, int d, cudaStream_t s) {
    FillArgs a{};
    a.seed = seed; a.kind = 2; a.rows = vocab; a.cols = d; a.d = d;
    fill(dtype, dst, a, s);
}

void synth_head(int dtype, void* dst, uint64_t seed, int e, float alpha, int vocab, int d,
                cudaStream_t s, int row0, int rows) {
    FillArgs a{};
    a.seed = seed; a.kind = 3; a.rows = rows > 0 ? rows : vocab; a.cols = d; a.d = d; a.exit_index = e;
    a.row0 = row0;
    a.scale = alpha; a.vocab = (uint32_t)vocab; a.pmul = synth::perm_mul((uint32_t)vocab);
    fill(dtype, dst, a, s);
}

}  // namespace eeb
