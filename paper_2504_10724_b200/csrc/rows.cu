// rows.cu — per-row kernels around the GEMMs: embedding gather, the fused
// split-K reduction + residual add + RMSNorm, the fused reduction + MLP
// activation, and the row gather used by survivor compaction.
//
// Fusing the split-K reduction into these consumers removes a launch per
// GEMM and produces the next GEMM's normalised bf16 input in the same pass
// over the row (the residual stream stays f32).
#include "kernels.h"

namespace eeb {

namespace {

constexpr int kRowThreads = 256;

// Block-wide sum (fixed tree => deterministic).
__device__ __forceinline__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = 0.f;
    if (warp == 0) {
        t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.f;
        t = warp_sum(t);
        if (lane == 0) red[0] = t;
    }
    __syncthreads();
    return red[0];
}

// x[i] (+)= sum_s part[s][i]; out1 = T(x * inv_rms * g1); out2 likewise with g2.
// When part is null x is taken as is (first layer after the embedding).
template <typename T>
__global__ void __launch_bounds__(kRowThreads)
    residual_norm_kernel(const float* __restrict__ part, int splits, int64_t split_stride,
                         const int* __restrict__ n_active, float* __restrict__ x, int d, float eps,
                         const float* __restrict__ g1, T* __restrict__ out1, const float* __restrict__ g2,
                         T* __restrict__ out2) {
    const int i = blockIdx.x;
    if (i >= *n_active) return;
    extern __shared__ float xs[];  // [d]
    __shared__ float red[32];
    float* row = x + (int64_t)i * d;
    float ss = 0.f;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        float v = row[c];
        if (part) {
            float y = 0.f;
            for (int s = 0; s < splits; ++s) y += part[s * split_stride + (int64_t)i * d + c];
            v += y;
            row[c] = v;
        }
        xs[c] = v;
        ss += v * v;
    }
    const float tot = block_sum(ss, red);
    const float inv = rsqrtf(tot / (float)d + eps);
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        const float v = xs[c] * inv;
        out1[(int64_t)i * d + c] = from_f32<T>(v * g1[c]);
        if (out2) out2[(int64_t)i * d + c] = from_f32<T>(v * g2[c]);
    }
}

template <typename T>
__global__ void act_kernel(const float* __restrict__ part, int splits, int64_t split_stride,
                           const int* __restrict__ n_active, int N, int swiglu, T* __restrict__ out) {
    const int n_out = swiglu ? N / 2 : N;
    const int64_t total = (int64_t)(*n_active) * n_out;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n_out), n = (int)(idx % n_out);
        if (swiglu) {
            float g = 0.f, u = 0.f;
            for (int s = 0; s < splits; ++s) {
                const float2 gu = *reinterpret_cast<const float2*>(part + s * split_stride + (int64_t)i * N + 2 * n);
                g += gu.x;
                u += gu.y;
            }
            out[idx] = from_f32<T>(g / (1.f + __expf(-g)) * u);
        } else {
            float y = 0.f;
            for (int s = 0; s < splits; ++s) y += part[s * split_stride + (int64_t)i * N + n];
            out[idx] = from_f32<T>(fmaxf(y, 0.f));
        }
    }
}

template <typename T>
__global__ void embed_kernel(const T* __restrict__ emb, const int* __restrict__ tok,
                             const int* __restrict__ slot_in, const int* __restrict__ pos_in, int batch, int d,
                             RowState st) {
    const int i = blockIdx.x;
    if (i >= batch) return;
    if (threadIdx.x == 0) {
        st.row_of[i] = i;
        st.slot[i] = slot_in[i];
        st.pos[i] = pos_in[i];
        if (i == 0) *st.n_active = batch;
    }
    const T* src = emb + (int64_t)tok[i] * d;
    float* dst = st.x + (int64_t)i * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) dst[c] = to_f32(src[c]);
}

__global__ void gather_rows_kernel(const float* __restrict__ x_cur, float* __restrict__ x_nxt,
                                   const uint16_t* __restrict__ h_cur, uint16_t* __restrict__ h_nxt, int h_words,
                                   const int* __restrict__ src, const int* __restrict__ n_active, int d) {
    const int j = blockIdx.x;
    if (j >= *n_active) return;
    const int i = src[j];
    const float4* s = reinterpret_cast<const float4*>(x_cur + (int64_t)i * d);
    float4* o = reinterpret_cast<float4*>(x_nxt + (int64_t)j * d);
    for (int c = threadIdx.x; c < d / 4; c += blockDim.x) o[c] = s[c];
    if (h_cur) {
        const uint4* hs = reinterpret_cast<const uint4*>(h_cur + (int64_t)i * h_words);
        uint4* ho = reinterpret_cast<uint4*>(h_nxt + (int64_t)j * h_words);
        for (int c = threadIdx.x; c < h_words / 8; c += blockDim.x) ho[c] = hs[c];
    }
}

}  // namespace

void launch_embed(int dtype, const void* emb, const int* tok, const int* slot_in, const int* pos_in,
                  int batch, int d, RowState st, cudaStream_t s) {
    if (dtype == 0)
        embed_kernel<float><<<batch, 256, 0, s>>>(static_cast<const float*>(emb), tok, slot_in, pos_in, batch, d,
                                                  st);
    else
        embed_kernel<__nv_bfloat16><<<batch, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(emb), tok, slot_in,
                                                          pos_in, batch, d, st);
    EEB_CHECK_LAUNCH();
}

void launch_residual_norm(int dtype, const float* part, int splits, int64_t split_stride, const int* n_active,
                          int max_rows, float* x, int d, float eps, const float* g1, void* out1, const float* g2,
                          void* out2, cudaStream_t s) {
    const size_t smem = (size_t)d * 4;
    if (dtype == 0) {
        EEB_CUDA(cudaFuncSetAttribute(residual_norm_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        residual_norm_kernel<float><<<max_rows, kRowThreads, smem, s>>>(
            part, splits, split_stride, n_active, x, d, eps, g1, static_cast<float*>(out1), g2,
            static_cast<float*>(out2));
    } else {
        EEB_CUDA(cudaFuncSetAttribute(residual_norm_kernel<__nv_bfloat16>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        residual_norm_kernel<__nv_bfloat16><<<max_rows, kRowThreads, smem, s>>>(
            part, splits, split_stride, n_active, x, d, eps, g1, static_cast<__nv_bfloat16*>(out1), g2,
            static_cast<__nv_bfloat16*>(out2));
    }
    EEB_CHECK_LAUNCH();
}

void launch_act(int dtype, const float* part, int splits, int64_t split_stride, const int* n_active, int max_rows,
                int N, bool swiglu, void* out, int num_sms, cudaStream_t s) {
    const int n_out = swiglu ? N / 2 : N;
    int64_t blocks = ((int64_t)max_rows * n_out + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    if (dtype == 0)
        act_kernel<float><<<(int)blocks, 256, 0, s>>>(part, splits, split_stride, n_active, N, swiglu ? 1 : 0,
                                                      static_cast<float*>(out));
    else
        act_kernel<__nv_bfloat16><<<(int)blocks, 256, 0, s>>>(part, splits, split_stride, n_active, N,
                                                              swiglu ? 1 : 0, static_cast<__nv_bfloat16*>(out));
    EEB_CHECK_LAUNCH();
}

void launch_gather_rows(const float* x_cur, float* x_nxt, const void* h_cur, void* h_nxt, int h_bytes_per_row,
                        const int* src, const int* n_active, int max_rows, int d, cudaStream_t s) {
    gather_rows_kernel<<<max_rows, 256, 0, s>>>(x_cur, x_nxt, static_cast<const uint16_t*>(h_cur),
                                                static_cast<uint16_t*>(h_nxt), h_bytes_per_row / 2, src, n_active,
                                                d);
    EEB_CHECK_LAUNCH();
}

}  // namespace eeb
