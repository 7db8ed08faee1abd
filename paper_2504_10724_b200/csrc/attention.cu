// attention.cu — fused RoPE + KV append + single-query decode attention.
//
// One CTA per (live row, KV head); the CTA handles the G = H / Hkv query
// heads that share the KV head (GQA).  KV layout per layer:
// [slot][kv_head][position][head_dim], so one (row, kv head) streams a
// contiguous [pos+1, hd] block of K and V — the bytes that bound this kernel
// (B·S·2·d_kv·bw per layer).
//
// Early-exit KV semantics: a position whose token left the network before
// this layer has no K/V here (kv_depth[slot][p] < layer) and is masked; the
// current position is always valid because it is written by this kernel
// (SURVEY §7 hard part 5).
#include "kernels.h"

namespace eeb {

namespace {

constexpr int kThreads = 128;
constexpr int kChunk = 128;   // positions per online-softmax chunk (one per thread)
constexpr int kMaxG = 8;
constexpr int kMaxHd = 128;

template <typename T>
__device__ __forceinline__ float dot_row(const T* __restrict__ k, const float* __restrict__ q, int hd) {
    constexpr int VEC = Vec16<T>::N;
    float s = 0.f;
    for (int j = 0; j < hd; j += VEC) {
        float kv[VEC];
        unpack16(*reinterpret_cast<const uint4*>(k + j), kv, (const T*)nullptr);
#pragma unroll
        for (int t = 0; t < VEC; ++t) s = fmaf(q[j + t], kv[t], s);
    }
    return s;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) attention_kernel(AttnArgs a) {
    const int i = blockIdx.x;
    if (i >= *a.n_active) return;
    const int g = blockIdx.y;
    const int H = a.n_heads, Hkv = a.n_kv_heads, hd = a.head_dim, G = H / Hkv;
    const int dq = H * hd, dkv = Hkv * hd, half = hd / 2;
    const int slot = a.slot[i], pos = a.pos[i];
    const float* row = a.qkv + (int64_t)i * (dq + 2 * dkv);

    __shared__ float q_s[kMaxG][kMaxHd];
    __shared__ float kn_s[kMaxHd], vn_s[kMaxHd];
    __shared__ float p_s[kMaxG][kChunk];
    __shared__ float red_s[kMaxG][kThreads / 32];
    __shared__ float m_s[kMaxG], l_s[kMaxG], scale_s[kMaxG];
    __shared__ float o_s[kThreads][kMaxG];

    const float* cs = a.rope_cos + (int64_t)pos * half;
    const float* sn = a.rope_sin + (int64_t)pos * half;
    const float qscale = rsqrtf((float)hd);
    // RoPE (rotate-half) on the group's queries and on the new key.
    for (int idx = threadIdx.x; idx < G * hd; idx += kThreads) {
        const int h = idx / hd, j = idx % hd;
        const float* q = row + (g * G + h) * hd;
        const int jj = j < half ? j : j - half;
        const float x0 = q[jj], x1 = q[jj + half];
        const float v = j < half ? x0 * cs[jj] - x1 * sn[jj] : x0 * sn[jj] + x1 * cs[jj];
        q_s[h][j] = v * qscale;
    }
    T* kc = static_cast<T*>(a.k_cache) + (((int64_t)slot * Hkv + g) * a.max_seq) * hd;
    T* vc = static_cast<T*>(a.v_cache) + (((int64_t)slot * Hkv + g) * a.max_seq) * hd;
    for (int j = threadIdx.x; j < hd; j += kThreads) {
        const float* k = row + dq + g * hd;
        const float* v = row + dq + dkv + g * hd;
        const int jj = j < half ? j : j - half;
        const float x0 = k[jj], x1 = k[jj + half];
        const float kr = j < half ? x0 * cs[jj] - x1 * sn[jj] : x0 * sn[jj] + x1 * cs[jj];
        const T kt = from_f32<T>(kr), vt = from_f32<T>(v[j]);
        kc[(int64_t)pos * hd + j] = kt;
        vc[(int64_t)pos * hd + j] = vt;
        kn_s[j] = to_f32(kt);
        vn_s[j] = to_f32(vt);
    }
    if (threadIdx.x < kMaxG) {
        m_s[threadIdx.x] = -INFINITY;
        l_s[threadIdx.x] = 0.f;
    }
    __syncthreads();

    const uint8_t* depth = a.kv_depth + (int64_t)slot * a.max_seq;
    // PV mapping: thread -> (dim j, position lane pl); kThreads / hd position lanes.
    const int lanes_pv = kThreads / hd;
    const int j_pv = threadIdx.x % hd, pl = threadIdx.x / hd;
    float acc[kMaxG];
#pragma unroll
    for (int h = 0; h < kMaxG; ++h) acc[h] = 0.f;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c0 = 0; c0 <= pos; c0 += kChunk) {
        const int p = c0 + threadIdx.x;
        const bool valid = p <= pos && (p == pos || depth[p] >= a.layer);
        float s[kMaxG];
#pragma unroll
        for (int h = 0; h < kMaxG; ++h) s[h] = -INFINITY;
        if (valid) {
            if (p == pos) {
                for (int h = 0; h < G; ++h) {
                    float t = 0.f;
                    for (int j = 0; j < hd; ++j) t = fmaf(q_s[h][j], kn_s[j], t);
                    s[h] = t;
                }
            } else {
                const T* krow = kc + (int64_t)p * hd;
                for (int h = 0; h < G; ++h) s[h] = dot_row<T>(krow, q_s[h], hd);
            }
        }
        // chunk max per head
        for (int h = 0; h < G; ++h) {
            const float m = warp_max(s[h]);
            if (lane == 0) red_s[h][warp] = m;
        }
        __syncthreads();
        if (threadIdx.x < G) {
            const int h = threadIdx.x;
            float m = red_s[h][0];
            for (int w = 1; w < kThreads / 32; ++w) m = fmaxf(m, red_s[h][w]);
            const float m_new = fmaxf(m_s[h], m);
            scale_s[h] = m_new == -INFINITY ? 1.f : __expf(m_s[h] - m_new);
            m_s[h] = m_new;
        }
        __syncthreads();
        for (int h = 0; h < G; ++h) {
            const float e = valid ? __expf(s[h] - m_s[h]) : 0.f;
            p_s[h][threadIdx.x] = e;
            const float ws = warp_sum(e);
            if (lane == 0) red_s[h][warp] = ws;
        }
        __syncthreads();
        if (threadIdx.x < G) {
            const int h = threadIdx.x;
            float t = 0.f;
            for (int w = 0; w < kThreads / 32; ++w) t += red_s[h][w];
            l_s[h] = l_s[h] * scale_s[h] + t;
        }
        // P·V for this chunk
        for (int h = 0; h < G; ++h) acc[h] *= scale_s[h];
        const int cn = min(kChunk, pos + 1 - c0);
        for (int t = pl; t < cn; t += lanes_pv) {
            const int pp = c0 + t;
            float vv;
            if (pp == pos) vv = vn_s[j_pv];
            else vv = to_f32(vc[(int64_t)pp * hd + j_pv]);
            for (int h = 0; h < G; ++h) acc[h] = fmaf(p_s[h][t], vv, acc[h]);
        }
        __syncthreads();
    }
    for (int h = 0; h < G; ++h) o_s[threadIdx.x][h] = acc[h];
    __syncthreads();
    T* out = static_cast<T*>(a.out) + (int64_t)i * dq;
    for (int idx = threadIdx.x; idx < G * hd; idx += kThreads) {
        const int h = idx / hd, j = idx % hd;
        float t = 0.f;
        for (int l = 0; l < lanes_pv; ++l) t += o_s[l * hd + j][h];
        out[(g * G + h) * hd + j] = from_f32<T>(t / l_s[h]);
    }
}

}  // namespace

void launch_attention(const AttnArgs& a, cudaStream_t s) {
    const int G = a.n_heads / a.n_kv_heads;
    if (G > kMaxG || a.head_dim > kMaxHd || a.head_dim % 16 != 0 || kThreads % a.head_dim != 0)
        throw Error(1, "attention: unsupported head geometry");
    dim3 grid(a.max_rows, a.n_kv_heads);
    if (a.dtype == 0) attention_kernel<float><<<grid, kThreads, 0, s>>>(a);
    else attention_kernel<__nv_bfloat16><<<grid, kThreads, 0, s>>>(a);
    EEB_CHECK_LAUNCH();
}

}  // namespace eeb
