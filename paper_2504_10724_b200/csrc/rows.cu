// rows.cu — per-row elementwise kernels: embedding gather, RMSNorm, row gather.
#include "kernels.h"

namespace eeb {

namespace {

template <typename T>
__global__ void embed_kernel(const T* __restrict__ emb, const int* __restrict__ tok,
                             const int* __restrict__ slot_in, const int* __restrict__ pos_in,
                             int batch, int d, RowState st) {
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

// One CTA per row.  Sum of squares in f32 with a fixed tree (deterministic).
template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x,
                                                      const float* __restrict__ gain,
                                                      const int* __restrict__ n_active, int d,
                                                      float eps, T* __restrict__ out) {
    const int i = blockIdx.x;
    if (i >= *n_active) return;
    const float* row = x + (int64_t)i * d;
    float ss = 0.f;
    for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
        const float4 v = *reinterpret_cast<const float4*>(row + c);
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    __shared__ float red[8];
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        v = warp_sum(v);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = rsqrtf(red[0] / (float)d + eps);
    T* o = out + (int64_t)i * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) o[c] = from_f32<T>(row[c] * inv * gain[c]);
}

__global__ void gather_rows_kernel(const float* __restrict__ x_cur, float* __restrict__ x_nxt,
                                   const int* __restrict__ src, const int* __restrict__ n_active,
                                   int d) {
    const int j = blockIdx.x;
    if (j >= *n_active) return;
    const float4* s = reinterpret_cast<const float4*>(x_cur + (int64_t)src[j] * d);
    float4* o = reinterpret_cast<float4*>(x_nxt + (int64_t)j * d);
    for (int c = threadIdx.x; c < d / 4; c += blockDim.x) o[c] = s[c];
}

}  // namespace

void launch_embed(int dtype, const void* emb, const int* tok, const int* slot_in, const int* pos_in,
                  int batch, int d, RowState st, cudaStream_t s) {
    if (dtype == 0)
        embed_kernel<float><<<batch, 256, 0, s>>>(static_cast<const float*>(emb), tok, slot_in,
                                                  pos_in, batch, d, st);
    else
        embed_kernel<__nv_bfloat16><<<batch, 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(emb), tok, slot_in, pos_in, batch, d, st);
    EEB_CHECK_LAUNCH();
}

void launch_rmsnorm(int dtype, const float* x, const float* gain, const int* n_active, int max_rows,
                    int d, float eps, void* out, cudaStream_t s) {
    if (dtype == 0)
        rmsnorm_kernel<float><<<max_rows, 256, 0, s>>>(x, gain, n_active, d, eps,
                                                       static_cast<float*>(out));
    else
        rmsnorm_kernel<__nv_bfloat16><<<max_rows, 256, 0, s>>>(
            x, gain, n_active, d, eps, static_cast<__nv_bfloat16*>(out));
    EEB_CHECK_LAUNCH();
}

void launch_gather_rows(const float* x_cur, float* x_nxt, const int* src, const int* n_active,
                        int max_rows, int d, cudaStream_t s) {
    gather_rows_kernel<<<max_rows, 256, 0, s>>>(x_cur, x_nxt, src, n_active, d);
    EEB_CHECK_LAUNCH();
}

}  // namespace eeb
