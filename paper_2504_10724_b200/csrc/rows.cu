// rows.cu — per-row kernels around the GEMMs: embedding gather, the fused
// split-K reduction + residual add + RMSNorm, the fused reduction + MLP
// activation, and the row gather used by survivor compaction.
//
// Fusing the split-K reduction into these consumers removes a launch per
// GEMM and produces the next GEMM's normalised bf16 input in the same pass
// over the row (the residual stream stays f32).
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

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
// A cluster of kClusterRow CTAs owns one row: each sums its column slice of the
// split-K planes (many independent loads in flight), the row's sum of squares
// is combined through distributed shared memory in rank order (deterministic),
// and each CTA normalises its slice.  part == null: x is taken as is.
constexpr int kClusterRow = 8;

template <typename T>
__global__ void __cluster_dims__(kClusterRow, 1, 1) __launch_bounds__(kRowThreads)
    residual_norm_kernel(const float* part, int splits, int64_t split_stride,
                         const int* n_active, float* x, int d, float eps,
                         const float* g1, T* out1, const float* g2,
                         T* out2) {
    pdl_launch_dependents();
    pdl_wait();
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int i = blockIdx.x / kClusterRow;
    const bool live = i < *n_active;  // uniform over the cluster
    __shared__ float red[32];
    __shared__ float ss_slice;
    const int per = d / kClusterRow;
    const int c0 = rank * per;
    float* row = x + (int64_t)i * d;
    constexpr int kMaxCols = 8;  // per thread: d <= 8 * 8 * 256
    float v[kMaxCols];
    float ss = 0.f;
    if (live) {
#pragma unroll
        for (int k = 0; k < kMaxCols; ++k) {
            const int c = c0 + threadIdx.x + k * kRowThreads;
            v[k] = 0.f;
            if (threadIdx.x + k * kRowThreads < per) {
                float xv = row[c];
                if (part) {
                    float y = 0.f;
                    for (int s = 0; s < splits; ++s) y += part[s * split_stride + (int64_t)i * d + c];
                    xv += y;
                    row[c] = xv;
                }
                v[k] = xv;
                ss += xv * xv;
            }
        }
    }
    ss = block_sum(ss, red);
    if (threadIdx.x == 0) ss_slice = ss;
    cluster.sync();
    float tot = 0.f;
    for (int r = 0; r < kClusterRow; ++r) tot += *cluster.map_shared_rank(&ss_slice, r);
    cluster.sync();  // keep every slice alive until all ranks have read it
    if (!live) return;
    const float inv = rsqrtf(tot / (float)d + eps);
#pragma unroll
    for (int k = 0; k < kMaxCols; ++k) {
        const int c = c0 + threadIdx.x + k * kRowThreads;
        if (threadIdx.x + k * kRowThreads < per) {
            const float nv = v[k] * inv;
            out1[(int64_t)i * d + c] = from_f32<T>(nv * g1[c]);
            if (out2) out2[(int64_t)i * d + c] = from_f32<T>(nv * g2[c]);
        }
    }
}

template <typename T>
__global__ void act_kernel(const float* part, int splits, int64_t split_stride,
                           const int* n_active, int N, int swiglu, T* out) {
    pdl_launch_dependents();
    pdl_wait();
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

__global__ void plane_sum_kernel(const float* part, int splits, int64_t split_stride, const int* n_active, int d,
                                 float* out) {
    pdl_launch_dependents();
    pdl_wait();
    const int64_t total = (int64_t)(*n_active) * d;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        float y = 0.f;
        for (int s = 0; s < splits; ++s) y += part[s * split_stride + idx];
        out[idx] = y;
    }
}

template <typename T>
__global__ void embed_kernel(const T* __restrict__ emb, const int* tok,
                             const int* slot_in, const int* pos_in, int batch, int d,
                             RowState st) {
    pdl_launch_dependents();
    pdl_wait();
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

__global__ void gather_rows_kernel(const float* x_cur, float* x_nxt,
                                   const uint16_t* h_cur, uint16_t* h_nxt, int h_words,
                                   const int* src, const int* n_active, int d) {
    pdl_launch_dependents();
    pdl_wait();
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
        launch_pdl(embed_kernel<float>, dim3(batch), dim3(256), 0, s, static_cast<const float*>(emb), tok, slot_in,
                   pos_in, batch, d, st);
    else
        launch_pdl(embed_kernel<__nv_bfloat16>, dim3(batch), dim3(256), 0, s,
                   static_cast<const __nv_bfloat16*>(emb), tok, slot_in, pos_in, batch, d, st);
    EEB_CHECK_LAUNCH();
}

void launch_residual_norm(int dtype, const float* part, int splits, int64_t split_stride, const int* n_active,
                          int max_rows, float* x, int d, float eps, const float* g1, void* out1, const float* g2,
                          void* out2, cudaStream_t s) {
    if (d % kClusterRow != 0 || d / kClusterRow > 8 * kRowThreads)
        throw Error(1, "residual_norm: d_model must be a multiple of 8 and at most 16384");
    const dim3 grid(max_rows * kClusterRow);
    if (dtype == 0)
        launch_pdl(residual_norm_kernel<float>, grid, dim3(kRowThreads), 0, s, part, splits, split_stride, n_active, x,
                   d, eps, g1, static_cast<float*>(out1), g2, static_cast<float*>(out2));
    else
        launch_pdl(residual_norm_kernel<__nv_bfloat16>, grid, dim3(kRowThreads), 0, s, part, splits, split_stride,
                   n_active, x, d, eps, g1, static_cast<__nv_bfloat16*>(out1), g2, static_cast<__nv_bfloat16*>(out2));
    EEB_CHECK_LAUNCH();
}

void launch_plane_sum(const float* part, int splits, int64_t split_stride, const int* n_active, int max_rows, int d,
                      float* out, int num_sms, cudaStream_t s) {
    int64_t blocks = ((int64_t)max_rows * d + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    launch_pdl(plane_sum_kernel, dim3((unsigned)blocks), dim3(256), 0, s, part, splits, split_stride, n_active, d, out);
    EEB_CHECK_LAUNCH();
}

void launch_act(int dtype, const float* part, int splits, int64_t split_stride, const int* n_active, int max_rows,
                int N, bool swiglu, void* out, int num_sms, cudaStream_t s) {
    const int n_out = swiglu ? N / 2 : N;
    int64_t blocks = ((int64_t)max_rows * n_out + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    if (dtype == 0)
        launch_pdl(act_kernel<float>, dim3((unsigned)blocks), dim3(256), 0, s, part, splits, split_stride, n_active, N,
                   swiglu ? 1 : 0, static_cast<float*>(out));
    else
        launch_pdl(act_kernel<__nv_bfloat16>, dim3((unsigned)blocks), dim3(256), 0, s, part, splits, split_stride,
                   n_active, N, swiglu ? 1 : 0, static_cast<__nv_bfloat16*>(out));
    EEB_CHECK_LAUNCH();
}

void launch_gather_rows(const float* x_cur, float* x_nxt, const void* h_cur, void* h_nxt, int h_bytes_per_row,
                        const int* src, const int* n_active, int max_rows, int d, cudaStream_t s) {
    launch_pdl(gather_rows_kernel, dim3(max_rows), dim3(256), 0, s, x_cur, x_nxt, static_cast<const uint16_t*>(h_cur),
               static_cast<uint16_t*>(h_nxt), h_bytes_per_row / 2, src, n_active, d);
    EEB_CHECK_LAUNCH();
}

}  // namespace eeb
