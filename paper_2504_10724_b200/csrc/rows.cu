// rows.cu — per-row kernels around the GEMMs: embedding gather, the fused
// split-K reduction + residual add + RMSNorm, the fused reduction + MLP
// activation, and the row gather used by survivor compaction.
//
// Fusing the split-K reduction into these consumers removes a launch per
// GEMM and produces the next GEMM's normalised bf16 input in the same pass
// over the row (the residual stream stays f32).
#include <algorithm>

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
// One CTA per row (no cluster: a cluster launch costs ~1.5 us more per kernel
// in the step's graph than the whole row's work, tools/micro/rows_bench.cu).
// A thread owns kV float4 column groups; the planes are read kBatch at a time
// into registers before they are added (in plane order, so the sum equals a
// sequential one): one L2 round trip per kBatch planes, not one per plane.
// The row's sum of squares is a fixed-tree block reduction (deterministic).
// part == null: x is taken as is.
constexpr int kBatch = 8;
constexpr int kNormThreads = 512;

template <typename T>
__device__ __forceinline__ void store4(T* dst, float4 v);
template <>
__device__ __forceinline__ void store4<float>(float* dst, float4 v) {
    *reinterpret_cast<float4*>(dst) = v;
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* dst, float4 v) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(dst) = u;
}
__device__ __forceinline__ void add4(float4& a, const float4 b) {
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}

template <typename T, int kV>
__global__ void __launch_bounds__(kNormThreads)
    residual_norm_kernel(Stamp stamp, const float* part, int splits, int64_t split_stride,
                         const int* n_active, float* x, int d, float eps,
                         const float* g1, T* out1, const float* g2,
                         T* out2, const void* pf, size_t pf_bytes) {
    StampScope stamp_scope(stamp);
    pdl_launch_dependents();
    // the norm gains are weights: in registers before the wait (one dependent
    // L2 round trip fewer after it)
    float4 gr1[kV], gr2[kV];
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        if (c < d) {
            gr1[k] = __ldg(reinterpret_cast<const float4*>(g1 + c));
            if (out2) gr2[k] = __ldg(reinterpret_cast<const float4*>(g2 + c));
        }
    }
    pdl_wait();
    stamp_waited(stamp);
    // the next GEMM's weights -> L2 while this latency-bound pass runs (after
    // the wait: the predecessor GEMM's own weight stream has ended)
    if (threadIdx.x < 32) l2_prefetch_share(pf, pf_bytes, threadIdx.x);
    const int i = blockIdx.x;
    if (i >= *n_active) return;
    __shared__ float red[32];
    float* row = x + (int64_t)i * d;
    float4 v[kV];
    float ss = 0.f;
    // wide rows with few planes (34B: 4 float4 groups x 4 planes per thread):
    // every load of the thread in flight at once, then the same in-order sums
    // (the general loop below issues one column group's loads at a time)
    constexpr int kP = 24 / kV;
    if (kV > 1 && part && splits <= kP) {
        float4 xs[kV], t[kV][kP];
#pragma unroll
        for (int k = 0; k < kV; ++k) {
            const int c = 4 * (threadIdx.x + k * blockDim.x);
            if (c < d) {
                xs[k] = *reinterpret_cast<const float4*>(row + c);
#pragma unroll
                for (int j = 0; j < kP; ++j)
                    if (j < splits) t[k][j] = __ldcg(reinterpret_cast<const float4*>(part + (int64_t)i * d + c + j * split_stride));
            }
        }
#pragma unroll
        for (int k = 0; k < kV; ++k) {
            const int c = 4 * (threadIdx.x + k * blockDim.x);
            v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c < d) {
                float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int j = 0; j < kP; ++j)
                    if (j < splits) add4(y, t[k][j]);
                add4(xs[k], y);
                *reinterpret_cast<float4*>(row + c) = xs[k];
                v[k] = xs[k];
                ss += xs[k].x * xs[k].x + xs[k].y * xs[k].y + xs[k].z * xs[k].z + xs[k].w * xs[k].w;
            }
        }
    } else
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < d) {
            float4 xv = *reinterpret_cast<const float4*>(row + c);
            if (part) {
                const float* src = part + (int64_t)i * d + c;
                float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
                // one group per thread (d <= 2048): all 16 planes of C2's O / down
                // GEMMs in one round trip (1.459 -> 1.450 ms/step); wider rows keep
                // 8 (registers)
                constexpr int kB = kV == 1 ? 16 : kBatch;
                for (int s0 = 0; s0 < splits; s0 += kB) {
                    float4 t[kB];
#pragma unroll
                    for (int j = 0; j < kB; ++j)
                        if (s0 + j < splits) t[j] = __ldcg(reinterpret_cast<const float4*>(src + (s0 + j) * split_stride));
#pragma unroll
                    for (int j = 0; j < kB; ++j)
                        if (s0 + j < splits) add4(y, t[j]);
                }
                add4(xv, y);
                *reinterpret_cast<float4*>(row + c) = xv;
            }
            v[k] = xv;
            ss += xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
        }
    }
    ss = block_sum(ss, red);
    const float inv = rsqrtf(ss / (float)d + eps);
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        if (c < d) {
            const float4 gg = gr1[k];
            const float4 nv = make_float4(v[k].x * inv, v[k].y * inv, v[k].z * inv, v[k].w * inv);
            store4<T>(out1 + (int64_t)i * d + c, make_float4(nv.x * gg.x, nv.y * gg.y, nv.z * gg.z, nv.w * gg.w));
            if (out2) {
                const float4 g = gr2[k];
                store4<T>(out2 + (int64_t)i * d + c, make_float4(nv.x * g.x, nv.y * g.y, nv.z * g.z, nv.w * g.w));
            }
        }
    }
}

template <typename T>
__global__ void act_kernel(Stamp stamp, const float* part, int splits, int64_t split_stride,
                           const int* n_active, int N, int swiglu, T* out) {
    StampScope stamp_scope(stamp);
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

__global__ void plane_sum_kernel(Stamp stamp, const float* part, int splits, int64_t split_stride, const int* n_active, int d,
                                 float* out) {
    StampScope stamp_scope(stamp);
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
__global__ void embed_kernel(Stamp stamp, const T* __restrict__ emb, const int* tok,
                             const int* slot_in, const int* pos_in, int batch, int d,
                             RowState st) {
    StampScope stamp_scope(stamp);
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

// Embedding gather fused with the first layer's RMSNorm (bf16 models): x =
// emb[tok], out = bf16(x * rsqrt(mean x^2 + eps) * g) — the same per-thread
// float4 groups and fixed-tree block sum as residual_norm_kernel (part = null),
// so the result equals the embed + norm pair bit for bit, one launch fewer.
template <int kV>
__global__ void __launch_bounds__(kNormThreads)
    embed_norm_kernel(Stamp stamp, const __nv_bfloat16* __restrict__ emb, const int* tok, const int* slot_in,
                      const int* pos_in, int batch, int d, RowState st, float eps, const float* g,
                      __nv_bfloat16* out) {
    StampScope stamp_scope(stamp);
    pdl_launch_dependents();
    float4 gr[kV];  // weights: before the wait
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        if (c < d) gr[k] = __ldg(reinterpret_cast<const float4*>(g + c));
    }
    pdl_wait();
    const int i = blockIdx.x;
    if (i >= batch) return;
    __shared__ float red[32];
    if (threadIdx.x == 0) {
        st.row_of[i] = i;
        st.slot[i] = slot_in[i];
        st.pos[i] = pos_in[i];
        if (i == 0) *st.n_active = batch;
    }
    const __nv_bfloat16* src = emb + (int64_t)tok[i] * d;
    float* row = st.x + (int64_t)i * d;
    float4 v[kV];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < d) {
            const uint2 u = *reinterpret_cast<const uint2*>(src + c);
            float4 xv;
            xv.x = __uint_as_float(u.x << 16);
            xv.y = __uint_as_float(u.x & 0xffff0000u);
            xv.z = __uint_as_float(u.y << 16);
            xv.w = __uint_as_float(u.y & 0xffff0000u);
            *reinterpret_cast<float4*>(row + c) = xv;
            v[k] = xv;
            ss += xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
        }
    }
    ss = block_sum(ss, red);
    const float inv = rsqrtf(ss / (float)d + eps);
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        if (c < d) {
            const float4 gg = gr[k];
            const float4 nv = make_float4(v[k].x * inv, v[k].y * inv, v[k].z * inv, v[k].w * inv);
            store4<__nv_bfloat16>(out + (int64_t)i * d + c,
                                  make_float4(nv.x * gg.x, nv.y * gg.y, nv.z * gg.z, nv.w * gg.w));
        }
    }
}

__global__ void gather_rows_kernel(Stamp stamp, const float* x_cur, float* x_nxt,
                                   const uint16_t* h_cur, uint16_t* h_nxt, int h_words,
                                   const int* src, const int* n_active, int d) {
    StampScope stamp_scope(stamp);
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


// ---- tensor-parallel exchange over peer memory (see kernels.h) ---------------
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Spin until *flag >= want.  A peer that never arrives (a rank that died or
// launched a different exchange sequence) traps after ~10 s instead of
// hanging the device.
__device__ __forceinline__ void px_wait(const uint32_t* flag, uint32_t want) {
    if ((int32_t)(ld_acquire_sys(flag) - want) >= 0) return;
    const unsigned long long t0 = gtimer();
    while ((int32_t)(ld_acquire_sys(flag) - want) < 0) {
        __nanosleep(64);
        if (gtimer() - t0 > 10000000000ull) {
            printf("eeb: tensor-parallel exchange timed out (flag %p want %u have %u)\n", flag, want,
                   ld_acquire_sys(flag));
            __trap();
        }
    }
}
__device__ __forceinline__ uint32_t* px_u32(const PxPeers& px, int rank, int64_t off) {
    return reinterpret_cast<uint32_t*>(px.base[rank] + off);
}

// One CTA per row (grid = the step's max rows, identical on every rank).
template <typename T, int kV>
__global__ void __launch_bounds__(kNormThreads)
    tp_norm_kernel(Stamp stamp, PxPeers px, int planes, int64_t plane_stride, const int* n_active, float* x, int d,
                   float eps, const float* g1, T* out1, const float* g2, T* out2) {
    StampScope stamp_scope(stamp);
    float4 gr1[kV], gr2[kV];  // weights: before the wait
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        if (c < d && out1) {
            gr1[k] = __ldg(reinterpret_cast<const float4*>(g1 + c));
            if (out2) gr2[k] = __ldg(reinterpret_cast<const float4*>(g2 + c));
        }
    }
    pdl_wait();  // this rank's partial planes are complete
    stamp_waited(stamp);
    const int i = blockIdx.x, me = px.rank, N = px.nranks;
    __shared__ float red[32];
    __shared__ uint32_t epoch_s;
    uint32_t* epoch_cell = px_u32(px, me, px.lay.epoch) + i;
    // 1. every rank's CTA i has arrived: its partial planes are complete
    if (threadIdx.x == 0) {
        const uint32_t e = *epoch_cell + 1;
        epoch_s = e;
        __threadfence_system();
        for (int p = 0; p < N; ++p)
            if (p != me) st_release_sys(px_u32(px, p, px.lay.arrive) + me * kPxMaxCtas + i, e);
        for (int p = 0; p < N; ++p)
            if (p != me) px_wait(px_u32(px, me, px.lay.arrive) + p * kPxMaxCtas + i, e);
    }
    __syncthreads();
    const uint32_t e = epoch_s;
    const int n = *n_active;
    const bool live = i < n;
    // 2. reduce-scatter: this rank sums its 1/N slice of row i over every
    // rank's planes (rank-major, then plane order) and stores the slice into
    // every rank's reduced row (all-gather by push)
    if (live) {
        const int q = d / 4, g0 = me * q / N, g1e = (me + 1) * q / N;
        for (int gi = g0 + (int)threadIdx.x; gi < g1e; gi += blockDim.x) {
            const int c = 4 * gi;
            float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int p = 0; p < N; ++p) {
                const float* src = reinterpret_cast<const float*>(px.base[p] + px.lay.planes) + (int64_t)i * d + c;
                for (int s0 = 0; s0 < planes; s0 += kBatch) {
                    float4 t[kBatch];
#pragma unroll
                    for (int j = 0; j < kBatch; ++j)
                        if (s0 + j < planes) t[j] = __ldcg(reinterpret_cast<const float4*>(src + (s0 + j) * plane_stride));
#pragma unroll
                    for (int j = 0; j < kBatch; ++j)
                        if (s0 + j < planes) add4(y, t[j]);
                }
            }
            for (int p = 0; p < N; ++p)
                __stcg(reinterpret_cast<float4*>(reinterpret_cast<float*>(px.base[p] + px.lay.red) + (int64_t)i * d + c), y);
        }
    }
    // 3. every rank's slice of row i has landed here
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int p = 0; p < N; ++p)
            if (p != me) st_release_sys(px_u32(px, p, px.lay.pushed) + me * kPxMaxCtas + i, e);
        for (int p = 0; p < N; ++p)
            if (p != me) px_wait(px_u32(px, me, px.lay.pushed) + p * kPxMaxCtas + i, e);
    }
    __syncthreads();
    float4 y[kV];
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        y[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (live && c < d)
            y[k] = __ldcg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(px.base[me] + px.lay.red) +
                                                          (int64_t)i * d + c));
    }
    if (threadIdx.x == 0) *epoch_cell = e;
    pdl_launch_dependents();
    if (!live) return;
    // x += sum; RMSNorm — as residual_norm_kernel
    float* row = x + (int64_t)i * d;
    float4 v[kV];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < d) {
            float4 xv = *reinterpret_cast<const float4*>(row + c);
            add4(xv, y[k]);
            *reinterpret_cast<float4*>(row + c) = xv;
            v[k] = xv;
            ss += xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
        }
    }
    ss = block_sum(ss, red);
    const float inv = rsqrtf(ss / (float)d + eps);
    if (!out1) return;
#pragma unroll
    for (int k = 0; k < kV; ++k) {
        const int c = 4 * (threadIdx.x + k * blockDim.x);
        if (c < d) {
            const float4 gg = gr1[k];
            const float4 nv = make_float4(v[k].x * inv, v[k].y * inv, v[k].z * inv, v[k].w * inv);
            store4<T>(out1 + (int64_t)i * d + c, make_float4(nv.x * gg.x, nv.y * gg.y, nv.z * gg.z, nv.w * gg.w));
            if (out2) {
                const float4 g = gr2[k];
                store4<T>(out2 + (int64_t)i * d + c, make_float4(nv.x * g.x, nv.y * g.y, nv.z * g.z, nv.w * g.w));
            }
        }
    }
}

// Pull-style all-gather: after every rank's CTA b arrived (its head partials
// are complete), CTA b copies its slice of every rank's head area into dst.
// A rank overwrites its head area only at its next exit head, i.e. after at
// least one tp_norm exchange, which every rank enters only once its previous
// kernels (this gather included) have finished.
__global__ void __launch_bounds__(256) px_gather_kernel(Stamp stamp, PxPeers px, int64_t region4, float4* dst) {
    StampScope stamp_scope(stamp);
    pdl_wait();
    stamp_waited(stamp);
    const int b = blockIdx.x, me = px.rank;
    __shared__ uint32_t epoch_s;
    uint32_t* epoch_cell = px_u32(px, me, px.lay.g_epoch) + b;
    if (threadIdx.x == 0) {
        const uint32_t e = *epoch_cell + 1;
        epoch_s = e;
        __threadfence_system();
        for (int p = 0; p < px.nranks; ++p)
            if (p != me) st_release_sys(px_u32(px, p, px.lay.g_arrive) + me * kPxGatherCtas + b, e);
        for (int p = 0; p < px.nranks; ++p)
            if (p != me) px_wait(px_u32(px, me, px.lay.g_arrive) + p * kPxGatherCtas + b, e);
    }
    __syncthreads();
    for (int p = 0; p < px.nranks; ++p) {
        const float4* src = reinterpret_cast<const float4*>(px.base[p] + px.lay.head);
        for (int64_t k = (int64_t)b * blockDim.x + threadIdx.x; k < region4; k += (int64_t)gridDim.x * blockDim.x)
            dst[p * region4 + k] = __ldcg(src + k);
    }
    if (threadIdx.x == 0) *epoch_cell = epoch_s;
    pdl_launch_dependents();
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

bool launch_embed_norm(int dtype, const void* emb, const int* tok, const int* slot_in, const int* pos_in, int batch,
                       int d, RowState st, float eps, const float* g, void* out, cudaStream_t s) {
    const int q = d / 4;
    if (dtype != 1 || d % 4 != 0 || q > 4 * kNormThreads) return false;
    const int kv = q <= kNormThreads ? 1 : (q <= 2 * kNormThreads ? 2 : 4);
    const dim3 grid(batch), block(std::max(32, std::min(kNormThreads, (q / kv + 31) / 32 * 32)));
    auto go = [&](auto kern) {
        launch_pdl(kern, grid, block, 0, s, static_cast<const __nv_bfloat16*>(emb), tok, slot_in, pos_in, batch, d, st,
                   eps, g, static_cast<__nv_bfloat16*>(out));
    };
    if (kv == 1) go(embed_norm_kernel<1>);
    else if (kv == 2) go(embed_norm_kernel<2>);
    else go(embed_norm_kernel<4>);
    EEB_CHECK_LAUNCH();
    return true;
}

// float4 groups per thread of the row kernels: the fewest that fit 512
// threads, or min_vec (prefill chunks of up to 1024 rows: 4 -> 128-thread CTAs,
// 16 resident per SM instead of 4, the whole chunk in one wave; the row sum's
// order follows the choice, so decode and prefill each keep one)
int norm_vec(int q, int min_vec) {
    int kv = q <= kNormThreads ? 1 : (q <= 2 * kNormThreads ? 2 : 4);
    while (kv < min_vec && kv < 4 && q / (2 * kv) >= 32) kv *= 2;
    return kv;
}

void launch_residual_norm(int dtype, const float* part, int splits, int64_t split_stride, const int* n_active,
                          int max_rows, float* x, int d, float eps, const float* g1, void* out1, const float* g2,
                          void* out2, cudaStream_t s, const void* pf, size_t pf_bytes, int min_vec) {
    const int q = d / 4;  // float4 groups per row
    if (d % 4 != 0 || q > 4 * kNormThreads)
        throw Error(1, "residual_norm: d_model must be a multiple of 4 and at most 8192");
    const int kv = norm_vec(q, min_vec);
    const dim3 grid(max_rows), block(std::max(32, std::min(kNormThreads, (q / kv + 31) / 32 * 32)));
    auto go = [&](auto kern, auto* o1, auto* o2) {
        launch_pdl(kern, grid, block, 0, s, part, splits, split_stride, n_active, x, d, eps, g1, o1, g2, o2, pf,
                   pf_bytes);
    };
    if (dtype == 0) {
        float* o1 = static_cast<float*>(out1);
        float* o2 = static_cast<float*>(out2);
        if (kv == 1) go(residual_norm_kernel<float, 1>, o1, o2);
        else if (kv == 2) go(residual_norm_kernel<float, 2>, o1, o2);
        else go(residual_norm_kernel<float, 4>, o1, o2);
    } else {
        __nv_bfloat16* o1 = static_cast<__nv_bfloat16*>(out1);
        __nv_bfloat16* o2 = static_cast<__nv_bfloat16*>(out2);
        if (kv == 1) go(residual_norm_kernel<__nv_bfloat16, 1>, o1, o2);
        else if (kv == 2) go(residual_norm_kernel<__nv_bfloat16, 2>, o1, o2);
        else go(residual_norm_kernel<__nv_bfloat16, 4>, o1, o2);
    }
    EEB_CHECK_LAUNCH();
}

void launch_tp_norm(int dtype, const PxPeers& px, int planes, int64_t plane_stride, const int* n_active, int max_rows,
                    float* x, int d, float eps, const float* g1, void* out1, const float* g2, void* out2,
                    cudaStream_t s, int min_vec) {
    const int q = d / 4;
    if (d % 4 != 0 || q > 4 * kNormThreads) throw Error(1, "tp_norm: d_model must be a multiple of 4 and at most 8192");
    if (max_rows > kPxMaxCtas || max_rows > px.lay.rows) throw Error(1, "tp_norm: more rows than the exchange buffer holds");
    if (px.nranks < 2 || px.nranks > kPxMaxRanks) throw Error(1, "tp_norm: bad rank count");
    const int kv = norm_vec(q, min_vec);
    const dim3 grid(max_rows), block(std::max(32, std::min(kNormThreads, (q / kv + 31) / 32 * 32)));
    auto go = [&](auto kern, auto* o1, auto* o2) {
        launch_pdl(kern, grid, block, 0, s, px, planes, plane_stride, n_active, x, d, eps, g1, o1, g2, o2);
    };
    if (dtype == 0) {
        float* o1 = static_cast<float*>(out1);
        float* o2 = static_cast<float*>(out2);
        if (kv == 1) go(tp_norm_kernel<float, 1>, o1, o2);
        else if (kv == 2) go(tp_norm_kernel<float, 2>, o1, o2);
        else go(tp_norm_kernel<float, 4>, o1, o2);
    } else {
        __nv_bfloat16* o1 = static_cast<__nv_bfloat16*>(out1);
        __nv_bfloat16* o2 = static_cast<__nv_bfloat16*>(out2);
        if (kv == 1) go(tp_norm_kernel<__nv_bfloat16, 1>, o1, o2);
        else if (kv == 2) go(tp_norm_kernel<__nv_bfloat16, 2>, o1, o2);
        else go(tp_norm_kernel<__nv_bfloat16, 4>, o1, o2);
    }
    EEB_CHECK_LAUNCH();
}

void launch_px_gather(const PxPeers& px, int64_t region, float* dst, cudaStream_t s) {
    if (region % 4 != 0 || region > px.lay.head_elems) throw Error(1, "px_gather: region does not fit the exchange buffer");
    const int64_t r4 = region / 4;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(kPxGatherCtas, (r4 + 255) / 256));
    launch_pdl(px_gather_kernel, dim3(grid), dim3(256), 0, s, px, r4, reinterpret_cast<float4*>(dst));
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
