// attention.cu — fused RoPE + KV append + single-query decode attention.
//
// One CTA per (live row, KV head); the CTA serves the G = H / Hkv query heads
// that share the KV head (GQA).  KV layout per layer:
// [slot][kv_head][position][head_dim], so the keys (and values) one CTA needs
// are one contiguous block: a single cp.async.bulk per chunk moves it into
// shared memory, with every byte of the chunk in flight at once (the bytes
// are what bound this kernel: B·S·2·d_kv·bw per layer).  Scores,
// the online softmax and P·V then run out of shared memory.
//
// Early-exit KV semantics: a position whose token left the network before
// this layer has no K/V here (kv_depth[slot][p] < layer) and is masked; the
// current position is always valid because this kernel writes it
// (SURVEY §7 hard part 5).
#include "kernels.h"

namespace eeb {

namespace {

constexpr int kThreads = 128;
constexpr int kMaxG = 8;
constexpr int kMaxHd = 128;
constexpr int kChunkBytes = 32 * 1024;  // K (or V) bytes staged per chunk

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

template <typename T>
__global__ void __launch_bounds__(kThreads) attention_kernel(AttnArgs a) {
    constexpr int VEC = Vec16<T>::N;  // elements per 16 B
    const int i = blockIdx.x;
    if (i >= *a.n_active) return;
    const int g = blockIdx.y;
    const int H = a.n_heads, Hkv = a.n_kv_heads, hd = a.head_dim, G = H / Hkv;
    const int dq = H * hd, dkv = Hkv * hd, half = hd / 2;
    const int slot = a.slot[i], pos = a.pos[i];
    const int C = kChunkBytes / (hd * (int)sizeof(T));  // positions per chunk
    const int64_t row_off = (int64_t)i * (dq + 2 * dkv);
    // q/k/v element = fixed-order sum of the QKV GEMM's split-K planes
    auto qkv = [&](int col) {
        float v = 0.f;
        for (int s = 0; s < a.splits; ++s) v += a.qkv[s * a.split_stride + row_off + col];
        return v;
    };

    extern __shared__ __align__(128) uint8_t smem[];
    T* ks = reinterpret_cast<T*>(smem);                          // [C][hd]
    T* vs = reinterpret_cast<T*>(smem + kChunkBytes);            // [C][hd]
    float* q_s = reinterpret_cast<float*>(smem + 2 * kChunkBytes);  // [G][hd]
    float* sc = q_s + G * hd;                                     // [G][C]
    __shared__ float m_s[kMaxG], l_s[kMaxG], scale_s[kMaxG];
    __shared__ float kn_s[kMaxHd], vn_s[kMaxHd];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t bar_a = smem_u32(&bar);

    T* kc = static_cast<T*>(a.k_cache) + (((int64_t)slot * Hkv + g) * a.max_seq) * hd;
    T* vc = static_cast<T*>(a.v_cache) + (((int64_t)slot * Hkv + g) * a.max_seq) * hd;
    const int n_chunks = pos / C + 1;

    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // first chunk's copy overlaps with the RoPE / append below
        const int n_copy = min(C, pos);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a),
                     "r"((uint32_t)(2 * n_copy * hd * sizeof(T)))
                     : "memory");
        if (n_copy > 0) {
            bulk_g2s(smem_u32(ks), kc, n_copy * hd * sizeof(T), bar_a);
            bulk_g2s(smem_u32(vs), vc, n_copy * hd * sizeof(T), bar_a);
        }
    }
    if (threadIdx.x < kMaxG) {
        m_s[threadIdx.x] = -INFINITY;
        l_s[threadIdx.x] = 0.f;
    }

    // RoPE (rotate-half) on the group's queries and on the new key.
    const float* cs = a.rope_cos + (int64_t)pos * half;
    const float* sn = a.rope_sin + (int64_t)pos * half;
    const float qscale = rsqrtf((float)hd);
    for (int idx = threadIdx.x; idx < G * hd; idx += kThreads) {
        const int h = idx / hd, j = idx % hd;
        const int q0 = (g * G + h) * hd;
        const int jj = j < half ? j : j - half;
        const float x0 = qkv(q0 + jj), x1 = qkv(q0 + jj + half);
        const float v = j < half ? x0 * cs[jj] - x1 * sn[jj] : x0 * sn[jj] + x1 * cs[jj];
        q_s[h * hd + j] = v * qscale;
    }
    for (int j = threadIdx.x; j < hd; j += kThreads) {
        const int k0 = dq + g * hd, v0 = dq + dkv + g * hd;
        const int jj = j < half ? j : j - half;
        const float x0 = qkv(k0 + jj), x1 = qkv(k0 + jj + half);
        const float kr = j < half ? x0 * cs[jj] - x1 * sn[jj] : x0 * sn[jj] + x1 * cs[jj];
        const T kt = from_f32<T>(kr), vt = from_f32<T>(qkv(v0 + j));
        kc[(int64_t)pos * hd + j] = kt;
        vc[(int64_t)pos * hd + j] = vt;
        kn_s[j] = to_f32(kt);
        vn_s[j] = to_f32(vt);
    }

    const uint8_t* depth = a.kv_depth + (int64_t)slot * a.max_seq;
    const int npg = kThreads / (hd / 2);        // P·V position groups
    const int dp = threadIdx.x % (hd / 2);       // dim pair
    const int pg = threadIdx.x / (hd / 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int vpr = hd / VEC;                    // 16-byte vectors per row
    float acc[kMaxG][2];
#pragma unroll
    for (int h = 0; h < kMaxG; ++h) acc[h][0] = acc[h][1] = 0.f;

    for (int ci = 0; ci < n_chunks; ++ci) {
        const int c0 = ci * C;
        const int cn = min(C, pos + 1 - c0);     // positions in this chunk (incl. pos if last)
        if (ci > 0 && threadIdx.x == 0) {
            const int n_copy = min(C, pos - c0);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a),
                         "r"((uint32_t)(2 * n_copy * hd * sizeof(T)))
                         : "memory");
            if (n_copy > 0) {
                bulk_g2s(smem_u32(ks), kc + (int64_t)c0 * hd, n_copy * hd * sizeof(T), bar_a);
                bulk_g2s(smem_u32(vs), vc + (int64_t)c0 * hd, n_copy * hd * sizeof(T), bar_a);
            }
        }
        __syncthreads();  // q_s / kn_s ready (first chunk)
        mbar_wait(bar_a, (uint32_t)(ci & 1));

        // scores: thread per position; 16-byte chunks read in a lane-rotated
        // order so each quarter-warp hits distinct banks.
        for (int t = threadIdx.x; t < cn; t += kThreads) {
            const int p = c0 + t;
            const bool valid = p == pos || depth[p] >= a.layer;
            for (int h = 0; h < G; ++h) {
                float s = -INFINITY;
                if (valid) {
                    s = 0.f;
                    if (p == pos) {
                        for (int j = 0; j < hd; ++j) s = fmaf(q_s[h * hd + j], kn_s[j], s);
                    } else {
                        const T* kr = ks + t * hd;
                        for (int u = 0; u < vpr; ++u) {
                            const int cidx = (u + lane) % vpr;
                            float kv[VEC];
                            unpack16(*reinterpret_cast<const uint4*>(kr + cidx * VEC), kv, (const T*)nullptr);
                            const float* qq = q_s + h * hd + cidx * VEC;
#pragma unroll
                            for (int e = 0; e < VEC; ++e) s = fmaf(qq[e], kv[e], s);
                        }
                    }
                }
                sc[h * C + t] = s;
            }
        }
        __syncthreads();
        // online softmax: warp w owns heads w, w+4, ...
        for (int h = warp; h < G; h += kThreads / 32) {
            float m = -INFINITY;
            for (int t = lane; t < cn; t += 32) m = fmaxf(m, sc[h * C + t]);
            m = warp_max(m);
            const float m_new = fmaxf(m_s[h], m);
            float sum = 0.f;
            for (int t = lane; t < cn; t += 32) {
                const float s = sc[h * C + t];
                const float e = s == -INFINITY ? 0.f : __expf(s - m_new);
                sc[h * C + t] = e;
                sum += e;
            }
            sum = warp_sum(sum);
            if (lane == 0) {
                const float scl = m_s[h] == -INFINITY ? 0.f : __expf(m_s[h] - m_new);
                scale_s[h] = scl;
                l_s[h] = l_s[h] * scl + sum;
                m_s[h] = m_new;
            }
        }
        __syncthreads();
        // P·V: thread = (dim pair, position group)
        for (int h = 0; h < G; ++h) {
            acc[h][0] *= scale_s[h];
            acc[h][1] *= scale_s[h];
        }
        for (int t = pg; t < cn; t += npg) {
            const int p = c0 + t;
            float v0, v1;
            if (p == pos) {
                v0 = vn_s[2 * dp];
                v1 = vn_s[2 * dp + 1];
            } else {
                v0 = to_f32(vs[t * hd + 2 * dp]);
                v1 = to_f32(vs[t * hd + 2 * dp + 1]);
            }
            for (int h = 0; h < G; ++h) {
                const float w = sc[h * C + t];
                acc[h][0] = fmaf(w, v0, acc[h][0]);
                acc[h][1] = fmaf(w, v1, acc[h][1]);
            }
        }
        __syncthreads();  // smem chunk free for the next copy
    }
    // reduce the position groups through (now free) score memory
    float* red = sc;  // [npg][G][hd]
    for (int h = 0; h < G; ++h) {
        red[(pg * G + h) * hd + 2 * dp] = acc[h][0];
        red[(pg * G + h) * hd + 2 * dp + 1] = acc[h][1];
    }
    __syncthreads();
    T* out = static_cast<T*>(a.out) + (int64_t)i * dq;
    for (int idx = threadIdx.x; idx < G * hd; idx += kThreads) {
        const int h = idx / hd, j = idx % hd;
        float t = 0.f;
        for (int q = 0; q < npg; ++q) t += red[(q * G + h) * hd + j];
        out[(g * G + h) * hd + j] = from_f32<T>(t / l_s[h]);
    }
}

}  // namespace

void launch_attention(const AttnArgs& a, cudaStream_t s) {
    const int G = a.n_heads / a.n_kv_heads;
    if (G > kMaxG || a.head_dim > kMaxHd || a.head_dim % 16 != 0 || kThreads % (a.head_dim / 2) != 0)
        throw Error(1, "attention: unsupported head geometry");
    const int esz = a.dtype == 0 ? 4 : 2;
    const int C = kChunkBytes / (a.head_dim * esz);
    const int npg = kThreads / (a.head_dim / 2);
    const size_t sc_floats = std::max((size_t)G * C, (size_t)npg * G * a.head_dim);
    const size_t smem = 2 * kChunkBytes + (size_t)G * a.head_dim * 4 + sc_floats * 4;
    dim3 grid(a.max_rows, a.n_kv_heads);
    if (a.dtype == 0) {
        EEB_CUDA(cudaFuncSetAttribute(attention_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attention_kernel<float><<<grid, kThreads, smem, s>>>(a);
    } else {
        EEB_CUDA(cudaFuncSetAttribute(attention_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        attention_kernel<__nv_bfloat16><<<grid, kThreads, smem, s>>>(a);
    }
    EEB_CHECK_LAUNCH();
}

}  // namespace eeb
