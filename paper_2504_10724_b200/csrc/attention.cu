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
#include <cuda.h>

#include <cstdlib>
#include <string>

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
__global__ void __launch_bounds__(kThreads) attention_kernel(Stamp stamp, AttnArgs a) {
    StampScope stamp_scope(stamp);
    constexpr int VEC = Vec16<T>::N;  // elements per 16 B
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.y;
    if (i >= *a.n_active) return;
    const int g = blockIdx.x;
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
        if (!a.kv_ready) {
            kc[(int64_t)pos * hd + j] = kt;
            vc[(int64_t)pos * hd + j] = vt;
        }
        kn_s[j] = to_f32(kt);
        vn_s[j] = to_f32(vt);
    }

    const uint8_t* depth = a.kv_depth + (int64_t)slot * a.max_seq;
    const int npg = kThreads / (hd / 2);        // P·V position groups (head_dim 80: 3, threads 120+ idle)
    const int dp = threadIdx.x % (hd / 2);       // dim pair
    const int pg = threadIdx.x / (hd / 2);
    const bool pv = pg < npg;
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
        for (int t = pg; pv && t < cn; t += npg) {
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
    for (int h = 0; pv && h < G; ++h) {
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


// ---------------------------------------------------------------------------
// bf16 path: flash-decode on the tensor cores.
//
// Q (G <= 8 heads, padded to the 16 rows of an m16n8k16 A operand) times K^T
// and P times V run as mma.sync tiles; K and V chunks arrive by TMA in
// 128-byte-swizzled [positions][64 dims] boxes so every ldmatrix is
// conflict-free.  Warp w owns position tiles w, w+4, ... with its own online
// softmax; the four warps are combined at the end (split-K style).
// ---------------------------------------------------------------------------
constexpr int kBoxRows = 32;    // positions per TMA box
constexpr int kMmaWarps = 4;

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t* r) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t* r) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// byte offset of (row, 16-byte chunk) inside a 128B-swizzled [rows][128 B] block
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
    return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

// CP: positions per chunk; NB: chunk buffers (2 = the next chunk's TMA is in
// flight while this one computes)
template <int HD, int CP, int NB, bool PAGED, int W = kMmaWarps>
__global__ void __launch_bounds__(W * 32, HD == 64 ? 20 / W : 1)  // hd 64: 5 x 4-warp CTAs/SM (register-limited)
    attention_mma_kernel(Stamp stamp, const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                         AttnArgs a) {
    StampScope stamp_scope(stamp);
    constexpr int CB = HD / 64;                    // 64-dim column blocks
    constexpr int NT = HD / 8;                     // 8-dim n-tiles of O
    constexpr int KS = HD / 16;                    // 16-dim k-steps of Q.K
    constexpr int TPW = CP / 8 / W;        // position tiles per warp per chunk
    constexpr uint32_t kBlockBytes = CP * 128;     // one column block of a chunk
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.y;
    if (i >= *a.n_active) return;
    const int g = blockIdx.x;
    const int H = a.n_heads, Hkv = a.n_kv_heads, G = H / Hkv;
    const int dq = H * HD, dkv = Hkv * HD, half = HD / 2;
    const int slot = a.slot[i], pos = a.pos[i];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (sbase - raw);
    // buffer b: K at sbase + b * 2 * CB * kBlockBytes, V right after ([CB][CP][128 B] each)
    constexpr uint32_t kBufBytes = 2 * CB * kBlockBytes;
    float* q_s = reinterpret_cast<float*>(base + NB * kBufBytes);  // [8][HD]
    __shared__ float kn_s[HD], vn_s[HD];
    __shared__ __align__(8) uint64_t bars[NB];

    const int64_t row_off = (int64_t)i * (dq + 2 * dkv);
    // Page of each position: the unpaged pool's table is the identity (page ==
    // slot, no load on the TMA's critical path); a paged pool's row for this
    // slot is read into smem once.
    // (a separate instantiation: the unpaged kernel keeps its registers)
    constexpr int kMaxPt = PAGED ? 64 : 1;
    __shared__ int pt_s[kMaxPt];
    const int PS = PAGED ? a.page_size : a.max_seq;
    if constexpr (PAGED) {
        for (int t = threadIdx.x; t < a.pages_per_seq && t < kMaxPt; t += blockDim.x)
            pt_s[t] = a.page_table[(int64_t)slot * a.pages_per_seq + t];
        __syncthreads();
    }
    auto page_of = [&](int p) { return PAGED ? pt_s[p / PS] : slot; };
    auto row_of = [&](int p) { return PAGED ? p % PS : p; };
    // the new position's K/V row
    const int64_t new_off = (((int64_t)page_of(pos) * Hkv + g) * PS + row_of(pos)) * HD;
    __nv_bfloat16* kc = static_cast<__nv_bfloat16*>(a.k_cache) + new_off;
    __nv_bfloat16* vc = static_cast<__nv_bfloat16*>(a.v_cache) + new_off;

    const int n_all = pos / CP + 1;  // chunks of this row
    // KV split z owns chunks [cb, ce) (possibly none); the one holding pos writes the new K/V
    const int S = a.kv_splits, z = blockIdx.z;
    const int per = (n_all + S - 1) / S;
    const int cb = min(n_all, z * per), ce = min(n_all, cb + per);
    const int n_chunks = ce - cb;
    const bool owns_pos = ce == n_all && n_chunks > 0;
    // thread 0: TMA positions [c0, c0+cn) of local chunk li (rounded up to whole boxes) into buffer li % NB
    auto issue = [&](int li) {
        const int ci = cb + li;
        const int c0 = ci * CP, buf = li % NB;
        const uint32_t k_s = sbase + buf * kBufBytes, v_s = k_s + CB * kBlockBytes;
        const uint32_t bar_a = smem_u32(&bars[buf]);
        const int n_load = min(CP, pos + 1 - c0);
        const int boxes = n_load > 0 ? (n_load + kBoxRows - 1) / kBoxRows : 0;
        const uint32_t bytes = (uint32_t)boxes * CB * kBoxRows * 128 * 2;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(bytes) : "memory");
        for (int b = 0; b < boxes; ++b) {
            const int p = c0 + b * kBoxRows;  // page_size is a multiple of the box
            const int zc = page_of(p) * Hkv + g;
            for (int cb = 0; cb < CB; ++cb) {
                const uint32_t off = cb * kBlockBytes + b * kBoxRows * 128;
                tma_3d(k_s + off, &kmap, bar_a, cb * 64, row_of(p), zc);
                tma_3d(v_s + off, &vmap, bar_a, cb * 64, row_of(p), zc);
            }
        }
    };
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
        for (int b = 0; b < NB; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[b])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int c = 0; c < NB && c < n_chunks; ++c) issue(c);
    }
    // Stage this CTA's q (G heads), k and v columns, summed over the QKV GEMM's
    // split-K planes, with every load in flight at once (float4, planes unrolled).
    float* raw_s = q_s + 8 * HD;  // [(G + 2) * HD]
    {
        const int nq4 = G * HD / 4, n4 = (G + 2) * HD / 4;
        const float* src = a.qkv + row_off;
        for (int v4 = threadIdx.x; v4 < n4; v4 += blockDim.x) {
            const int col = v4 < nq4 ? g * G * HD + 4 * v4
                          : (v4 < nq4 + HD / 4 ? dq + g * HD + 4 * (v4 - nq4) : dq + dkv + g * HD + 4 * (v4 - nq4 - HD / 4));
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int sp = 0; sp < 16; ++sp) {
                if (sp < a.splits) {
                    const float4 t = *reinterpret_cast<const float4*>(src + sp * a.split_stride + col);
                    acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
                }
            }
            *reinterpret_cast<float4*>(raw_s + 4 * v4) = acc;
        }
    }
    // RoPE row and the KV-depth bytes of the positions, fetched in the same
    // latency window as the planes (not as dependent global loads later).
    __shared__ float cs[HD / 2], sn[HD / 2];
    // KV depth bytes of every position (all chunks, not only the first: a
    // global read inside the score loop stalls on long scoreboard)
    constexpr int kDep = CP > 1024 ? CP : 1024;
    __shared__ uint8_t dep_s[kDep];
    for (int t = threadIdx.x; t < half; t += blockDim.x) {
        cs[t] = a.rope_cos[(int64_t)pos * half + t];
        sn[t] = a.rope_sin[(int64_t)pos * half + t];
    }
    {
        const uint8_t* dsrc = a.kv_depth + (int64_t)slot * a.max_seq;
        for (int t = threadIdx.x; t < kDep && t <= pos; t += blockDim.x) dep_s[t] = dsrc[t];
    }
    __syncthreads();
    // RoPE: queries (scaled) into q_s, the new key/value into the cache and kn_s / vn_s.
    const float qscale = rsqrtf((float)HD);
    for (int idx = threadIdx.x; idx < 8 * HD; idx += blockDim.x) {
        const int h = idx / HD, j = idx % HD;
        float v = 0.f;
        if (h < G) {
            const float* q = raw_s + h * HD;
            const int jj = j < half ? j : j - half;
            const float x0 = q[jj], x1 = q[jj + half];
            v = (j < half ? x0 * cs[jj] - x1 * sn[jj] : x0 * sn[jj] + x1 * cs[jj]) * qscale;
        }
        q_s[h * HD + j] = v;
    }
    for (int j = threadIdx.x; j < HD; j += blockDim.x) {
        const float* k = raw_s + G * HD;
        const float* vv = raw_s + (G + 1) * HD;
        const int jj = j < half ? j : j - half;
        const float x0 = k[jj], x1 = k[jj + half];
        const float kr = j < half ? x0 * cs[jj] - x1 * sn[jj] : x0 * sn[jj] + x1 * cs[jj];
        const __nv_bfloat16 kt = __float2bfloat16_rn(kr), vt = __float2bfloat16_rn(vv[j]);
        if (!a.kv_ready && owns_pos) {
            kc[j] = kt;
            vc[j] = vt;
        }
        kn_s[j] = __bfloat162float(kt);
        vn_s[j] = __bfloat162float(vt);
    }
    __syncthreads();
    // Q as m16n8k16 A fragments: rows = heads (lane/4), rows 8..15 are zero.
    const int h = lane >> 2, kq = (lane & 3) * 2;
    uint32_t qa[KS][4];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
        qa[k][0] = pack_bf16(q_s[h * HD + 16 * k + kq], q_s[h * HD + 16 * k + kq + 1]);
        qa[k][1] = 0u;
        qa[k][2] = pack_bf16(q_s[h * HD + 16 * k + 8 + kq], q_s[h * HD + 16 * k + 8 + kq + 1]);
        qa[k][3] = 0u;
    }
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    const uint8_t* depth = a.kv_depth + (int64_t)slot * a.max_seq;

    for (int li = 0; li < n_chunks; ++li) {
        const int ci = cb + li;
        const int c0 = ci * CP;
        const int cn = min(CP, pos + 1 - c0);
        const int buf = li % NB;
        const uint32_t k_s = sbase + buf * kBufBytes, v_s = k_s + CB * kBlockBytes;
        if (NB == 1 && li > 0) {
            __syncthreads();  // everyone is done with the previous chunk
            if (threadIdx.x == 0) issue(li);
        }
        mbar_wait(smem_u32(&bars[buf]), (uint32_t)((li / NB) & 1));
        if (!a.kv_ready && pos < c0 + CP) {  // the new position lives in this chunk: write it (swizzled)
            const int r = pos - c0;
            uint8_t* bb = base + buf * kBufBytes;
            for (int j = threadIdx.x; j < HD; j += blockDim.x) {
                const uint32_t off = (j / 64) * kBlockBytes + swz(r, (j % 64) / 8) + (j % 8) * 2;
                *reinterpret_cast<__nv_bfloat16*>(bb + off) = __float2bfloat16_rn(kn_s[j]);
                *reinterpret_cast<__nv_bfloat16*>(bb + CB * kBlockBytes + off) = __float2bfloat16_rn(vn_s[j]);
            }
        }
        __syncthreads();
        // NB >= 2: everyone is past chunk li-1, so its buffer takes chunk li-1+NB
        // while this chunk computes
        if (NB >= 2 && threadIdx.x == 0 && li >= 1 && li - 1 + NB < n_chunks) issue(li - 1 + NB);
        const int n_tiles = (cn + 7) / 8;
        // scores for this warp's tiles (C fragment: row h, positions kq, kq+1)
        float sc[TPW][2];
        int my_tiles = 0;
        float cmax = -INFINITY;
#pragma unroll
        for (int tt = 0; tt < TPW; ++tt) {
            const int t = warp + tt * W;
            sc[tt][0] = sc[tt][1] = -INFINITY;
            if (t >= n_tiles) continue;
            my_tiles = tt + 1;
            float c[4] = {0.f, 0.f, 0.f, 0.f};
            const int row = t * 8 + (lane & 7);
#pragma unroll
            for (int k2 = 0; k2 < KS; k2 += 2) {
                // matrices: (k-step k2 lo, hi), (k-step k2+1 lo, hi)
                const int mi = lane >> 3;
                const int dim = 16 * (k2 + (mi >> 1)) + 8 * (mi & 1);
                uint32_t b[4];
                ldsm_x4(k_s + (dim / 64) * kBlockBytes + swz(row, (dim % 64) / 8), b);
                mma_bf16(c, qa[k2], b[0], b[1]);
                mma_bf16(c, qa[k2 + 1], b[2], b[3]);
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int p = c0 + t * 8 + kq + e;
                const bool valid = h < G && p <= pos && (p == pos || (p < kDep ? dep_s[p] : depth[p]) >= a.layer);
                sc[tt][e] = valid ? c[e] : -INFINITY;
                cmax = fmaxf(cmax, sc[tt][e]);
            }
        }
        // online softmax per (warp, head): reduce over the 4 lanes of a head
        cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, 1));
        cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, 2));
        const float m_new = fmaxf(m_run, cmax);
        const float scale = m_new == -INFINITY ? 1.f : __expf(m_run - m_new);
        float psum = 0.f;
#pragma unroll
        for (int tt = 0; tt < TPW; ++tt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float p = sc[tt][e] == -INFINITY ? 0.f : __expf(sc[tt][e] - m_new);
                sc[tt][e] = p;
                psum += p;
            }
        psum += __shfl_xor_sync(0xffffffffu, psum, 1);
        psum += __shfl_xor_sync(0xffffffffu, psum, 2);
        l_run = l_run * scale + psum;
        m_run = m_new;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            o[n][0] *= scale;
            o[n][1] *= scale;
        }
        // P.V over tile pairs (tiles of one pair need not be adjacent positions)
#pragma unroll
        for (int tt = 0; tt < TPW; tt += 2) {
            if (tt >= my_tiles) break;
            const int ta = warp + tt * W;
            const bool has_b = tt + 1 < my_tiles;
            const int tb = has_b ? ta + W : ta;  // pad with a loaded tile, P = 0
            uint32_t pa[4];
            pa[0] = pack_bf16(sc[tt][0], sc[tt][1]);
            pa[1] = 0u;
            pa[2] = has_b ? pack_bf16(sc[tt + 1][0], sc[tt + 1][1]) : 0u;
            pa[3] = 0u;
            const int mi = lane >> 3;
            const int row = ((mi & 1) ? tb : ta) * 8 + (lane & 7);
#pragma unroll
            for (int n = 0; n < NT; n += 2) {
                const int dim = 8 * (n + (mi >> 1));
                uint32_t b[4];
                ldsm_x4_t(v_s + (dim / 64) * kBlockBytes + swz(row, (dim % 64) / 8), b);
                mma_bf16(o[n], pa, b[0], b[1]);
                mma_bf16(o[n + 1], pa, b[2], b[3]);
            }
        }
    }
    // combine the four warps: O = sum_w e^(m_w - M) O_w / sum_w e^(m_w - M) l_w
    __syncthreads();
    float* comb = reinterpret_cast<float*>(base);  // reuse the K/V chunk memory
    float* ml = comb + W * 8 * HD;          // [warp][head][2]
    if (h < G) {
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            comb[(warp * 8 + h) * HD + n * 8 + kq] = o[n][0];
            comb[(warp * 8 + h) * HD + n * 8 + kq + 1] = o[n][1];
        }
        if ((lane & 3) == 0) {
            ml[(warp * 8 + h) * 2] = m_run;
            ml[(warp * 8 + h) * 2 + 1] = l_run;
        }
    }
    __syncthreads();
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.out) + (int64_t)i * dq;
    // this CTA's partial per head: (O unnormalised w.r.t. its max M, M, l)
    float* part = S > 1 ? a.kv_part + ((int64_t)(i * Hkv + g) * S) * (8 * (HD + 2)) : nullptr;
    for (int idx = threadIdx.x; idx < G * HD; idx += blockDim.x) {
        const int hh = idx / HD, j = idx % HD;
        float M = -INFINITY;
        for (int w = 0; w < W; ++w) M = fmaxf(M, ml[(w * 8 + hh) * 2]);
        float num = 0.f, den = 0.f;
        for (int w = 0; w < W; ++w) {
            const float mw = ml[(w * 8 + hh) * 2];
            const float f = mw == -INFINITY ? 0.f : __expf(mw - M);
            num += f * comb[(w * 8 + hh) * HD + j];
            den += f * ml[(w * 8 + hh) * 2 + 1];
        }
        if (S == 1) {
            out[(g * G + hh) * HD + j] = __float2bfloat16_rn(num / den);
        } else {
            float* pz = part + (int64_t)z * (8 * (HD + 2)) + hh * (HD + 2);
            pz[j] = num;
            if (j == 0) {
                pz[HD] = M;
                pz[HD + 1] = den;
            }
        }
    }
    if (S == 1) return;
    __threadfence();
    __syncthreads();
    __shared__ int last_s;
    if (threadIdx.x == 0) last_s = atomicAdd(a.kv_ticket + i * Hkv + g, 1) == S - 1;
    __syncthreads();
    if (!last_s) return;
    __threadfence();
    // last split: combine the S partials in split order (deterministic)
    for (int idx = threadIdx.x; idx < G * HD; idx += blockDim.x) {
        const int hh = idx / HD, j = idx % HD;
        float M = -INFINITY;
        for (int q = 0; q < S; ++q) M = fmaxf(M, __ldcg(part + (int64_t)q * (8 * (HD + 2)) + hh * (HD + 2) + HD));
        float num = 0.f, den = 0.f;
        for (int q = 0; q < S; ++q) {
            const float* pq = part + (int64_t)q * (8 * (HD + 2)) + hh * (HD + 2);
            const float mq = __ldcg(pq + HD);
            const float f = mq == -INFINITY ? 0.f : __expf(mq - M);
            num += f * __ldcg(pq + j);
            den += f * __ldcg(pq + HD + 1);
        }
        out[(g * G + hh) * HD + j] = __float2bfloat16_rn(num / den);
    }
    if (threadIdx.x == 0) a.kv_ticket[i * Hkv + g] = 0;  // all splits arrived: ready for the next launch
}

// ---------------------------------------------------------------------------
// Pipelined variant: a CTA walks work items (row, kv-head) with a grid
// stride, and the K/V chunks of consecutive items stream through NBUF
// shared-memory buffers, so the TMA for the next item is in flight while the
// current one computes (the one-item-per-CTA kernel above exposes a full
// HBM latency per item; C2 has 2048 items of only ~45 KB each).  Chunks are
// smaller (32 KB of K+V) so three CTAs share an SM and one CTA's prologue
// (split-K plane sum, RoPE, KV append) overlaps the others' loads.
// ---------------------------------------------------------------------------
template <int HD>
struct PipeCfg {
    static constexpr int CB = HD / 64;
    static constexpr int CP = HD == 64 ? 128 : 64;           // positions per chunk
    static constexpr uint32_t kBlockBytes = CP * 128;        // one 64-dim column block
    static constexpr uint32_t kBufBytes = 2 * CB * kBlockBytes;  // K + V of one chunk
    static constexpr int NBUF = 2;
    static constexpr int NW = HD == 64 ? 8 : 4;  // warps: positions of a chunk split NW ways
};

// Shared-memory plan of the pipelined kernel (host and device agree).
template <int HD>
struct PipeSmem {
    int n4, pf_floats, pf_bytes;
    bool use_pf;
    size_t q_off, raw_off, pf_off, pos_off, total;
    __host__ __device__ PipeSmem(int G, int splits, int max_rows) {
        n4 = (G + 2) * HD / 4;
        pf_floats = splits * n4 * 4 + HD;  // split-K planes of q/k/v + the RoPE cos/sin halves
        pf_bytes = pf_floats * 4;
        use_pf = pf_bytes <= 16 * 1024;
        q_off = (size_t)PipeCfg<HD>::NBUF * PipeCfg<HD>::kBufBytes;
        raw_off = q_off + 8 * HD * 4;
        pf_off = raw_off + (size_t)(G + 2) * HD * 4;
        pos_off = pf_off + (use_pf ? 2 * (size_t)pf_bytes : 0);
        total = pos_off + 2 * (size_t)max_rows * 4;
    }
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int HD>
__global__ void __launch_bounds__(PipeCfg<HD>::NW * 32, 2)
    attention_pipe_kernel(Stamp stamp, const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                          AttnArgs a) {
    StampScope stamp_scope(stamp);
    using C = PipeCfg<HD>;
    constexpr int CB = C::CB, CP = C::CP, NBUF = C::NBUF, NW = C::NW;
    constexpr uint32_t kBlockBytes = C::kBlockBytes, kBufBytes = C::kBufBytes;
    constexpr int NT = HD / 8, KS = HD / 16, TPW = CP / 8 / NW;
    static_assert(CP <= C::NW * 32, "one depth byte per thread per chunk");
    pdl_launch_dependents();
    pdl_wait();
    const int H = a.n_heads, Hkv = a.n_kv_heads, G = H / Hkv;
    const int dq = H * HD, dkv = Hkv * HD, half = HD / 2;
    const int n_rows = *a.n_active;
    const int n_items = n_rows * Hkv;
    if ((int)blockIdx.x >= n_items) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const PipeSmem<HD> L(G, a.splits, a.max_rows);

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (sbase - raw);
    float* q_s = reinterpret_cast<float*>(base + L.q_off);      // [8][HD]
    float* raw_s = reinterpret_cast<float*>(base + L.raw_off);  // [(G + 2)][HD]
    float* pf = reinterpret_cast<float*>(base + L.pf_off);      // [2][pf_floats]
    int* pos_s = reinterpret_cast<int*>(base + L.pos_off);      // [rows]
    int* slot_s = pos_s + a.max_rows;
    __shared__ float kn_s[HD], vn_s[HD], cos_s[HD / 2], sin_s[HD / 2];
    __shared__ uint8_t dep_s[CP];
    __shared__ __align__(8) uint64_t bars[NBUF];

    for (int r = threadIdx.x; r < n_rows; r += blockDim.x) {
        pos_s[r] = a.pos[r];
        slot_s[r] = a.slot[r];
    }
    __syncthreads();

    auto n_chunks_of = [&](int item) { return pos_s[item / Hkv] / CP + 1; };
    auto issue = [&](int item, int chunk, int buf) {  // thread 0
        const int i = item / Hkv, g = item % Hkv;
        const int pos = pos_s[i], zc = slot_s[i] * Hkv + g;
        const int c0 = chunk * CP;
        const int n_load = min(CP, pos + 1 - c0);
        const int boxes = (n_load + kBoxRows - 1) / kBoxRows;
        const uint32_t bar = smem_u32(&bars[buf]);
        const uint32_t k_s = sbase + buf * kBufBytes, v_s = k_s + CB * kBlockBytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)boxes * CB * kBoxRows * 128 * 2)
                     : "memory");
        for (int b = 0; b < boxes; ++b)
            for (int cb = 0; cb < CB; ++cb) {
                const uint32_t off = cb * kBlockBytes + b * kBoxRows * 128;
                tma_3d(k_s + off, &kmap, bar, cb * 64, c0 + b * kBoxRows, zc);
                tma_3d(v_s + off, &vmap, bar, cb * 64, c0 + b * kBoxRows, zc);
            }
    };
    int is_item = blockIdx.x, is_chunk = 0;  // TMA issue cursor (thread 0)
    auto issue_next = [&](int buf) {
        if (is_item >= n_items) return;
        issue(is_item, is_chunk, buf);
        if (++is_chunk == n_chunks_of(is_item)) {
            is_chunk = 0;
            is_item += gridDim.x;
        }
    };
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
        for (int b = 0; b < NBUF; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[b])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int b = 0; b < NBUF; ++b) issue_next(b);
    }
    // column of the fused QKV row for float4 v4 of item (g): q heads, then k, then v
    auto col_of = [&](int v4, int g) {
        const int nq4 = G * HD / 4;
        return v4 < nq4 ? g * G * HD + 4 * v4
             : (v4 < nq4 + HD / 4 ? dq + g * HD + 4 * (v4 - nq4) : dq + dkv + g * HD + 4 * (v4 - nq4 - HD / 4));
    };
    // async prefetch of an item's q/k/v planes and RoPE row into pf[buf]
    auto prefetch = [&](int item, int buf) {
        if (item < n_items) {
            const int i = item / Hkv, g = item % Hkv;
            const float* src = a.qkv + (int64_t)i * (dq + 2 * dkv);
            float* dst = pf + (size_t)buf * L.pf_floats;
            for (int v4 = threadIdx.x; v4 < L.n4; v4 += blockDim.x) {
                const int col = col_of(v4, g);
                for (int sp = 0; sp < a.splits; ++sp)
                    cp_async16(dst + ((size_t)sp * L.n4 + v4) * 4, src + sp * a.split_stride + col);
            }
            const int pos = pos_s[i];
            for (int t = threadIdx.x; t < HD / 4; t += blockDim.x) {  // cos then sin, half floats each
                const float* r = t < HD / 8 ? a.rope_cos + (int64_t)pos * half + 4 * t
                                            : a.rope_sin + (int64_t)pos * half + 4 * (t - HD / 8);
                cp_async16(dst + (size_t)a.splits * L.n4 * 4 + 4 * t, r);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // depth byte of the next chunk in this CTA's walk, held in a register
    int dp_item = blockIdx.x, dp_chunk = 0;
    uint8_t dep_reg = 0;
    auto load_dep = [&]() {
        if (dp_item < n_items) {
            const int i = dp_item / Hkv;
            const int pos = pos_s[i], c0 = dp_chunk * CP;
            if ((int)threadIdx.x < min(CP, pos + 1 - c0))
                dep_reg = a.kv_depth[(int64_t)slot_s[i] * a.max_seq + c0 + threadIdx.x];
            if (++dp_chunk == pos / CP + 1) {
                dp_chunk = 0;
                dp_item += gridDim.x;
            }
        }
    };
    load_dep();
    if (L.use_pf) prefetch(blockIdx.x, 0);

    const int h = lane >> 2, kq = (lane & 3) * 2;
    const float qscale = rsqrtf((float)HD);
    uint32_t seq = 0;  // consumer's position in the TMA load sequence
    int it = 0;        // items processed by this CTA
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        const int i = item / Hkv, g = item % Hkv;
        const int slot = slot_s[i], pos = pos_s[i];
        __nv_bfloat16* kc = static_cast<__nv_bfloat16*>(a.k_cache) + (((int64_t)slot * Hkv + g) * a.max_seq) * HD;
        __nv_bfloat16* vc = static_cast<__nv_bfloat16*>(a.v_cache) + (((int64_t)slot * Hkv + g) * a.max_seq) * HD;
        // q (G heads), k, v of this item: fixed-order sum of the split-K planes
        if (L.use_pf) {
            prefetch(item + gridDim.x, (it + 1) & 1);  // next item's planes fly while this one computes
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncthreads();  // every thread's copies (the RoPE rows are read across threads)
            const float* src = pf + (size_t)(it & 1) * L.pf_floats;
            for (int v4 = threadIdx.x; v4 < L.n4; v4 += blockDim.x) {
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int sp = 0; sp < a.splits; ++sp) {
                    const float4 t = *reinterpret_cast<const float4*>(src + ((size_t)sp * L.n4 + v4) * 4);
                    acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
                }
                *reinterpret_cast<float4*>(raw_s + 4 * v4) = acc;
            }
            for (int t = threadIdx.x; t < HD; t += blockDim.x) {
                const float v = src[(size_t)a.splits * L.n4 * 4 + t];
                if (t < half) cos_s[t] = v;
                else sin_s[t - half] = v;
            }
        } else {
            const float* src = a.qkv + (int64_t)i * (dq + 2 * dkv);
            for (int v4 = threadIdx.x; v4 < L.n4; v4 += blockDim.x) {
                const int col = col_of(v4, g);
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int sp = 0; sp < 16; ++sp) {
                    if (sp < a.splits) {
                        const float4 t = *reinterpret_cast<const float4*>(src + sp * a.split_stride + col);
                        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
                    }
                }
                *reinterpret_cast<float4*>(raw_s + 4 * v4) = acc;
            }
            for (int t = threadIdx.x; t < half; t += blockDim.x) {
                cos_s[t] = a.rope_cos[(int64_t)pos * half + t];
                sin_s[t] = a.rope_sin[(int64_t)pos * half + t];
            }
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < 8 * HD; idx += blockDim.x) {
            const int hh = idx / HD, j = idx % HD;
            float v = 0.f;
            if (hh < G) {
                const float* q = raw_s + hh * HD;
                const int jj = j < half ? j : j - half;
                const float x0 = q[jj], x1 = q[jj + half];
                v = (j < half ? x0 * cos_s[jj] - x1 * sin_s[jj] : x0 * sin_s[jj] + x1 * cos_s[jj]) * qscale;
            }
            q_s[hh * HD + j] = v;
        }
        for (int j = threadIdx.x; j < HD; j += blockDim.x) {
            const float* k = raw_s + G * HD;
            const float* vv = raw_s + (G + 1) * HD;
            const int jj = j < half ? j : j - half;
            const float x0 = k[jj], x1 = k[jj + half];
            const float kr = j < half ? x0 * cos_s[jj] - x1 * sin_s[jj] : x0 * sin_s[jj] + x1 * cos_s[jj];
            const __nv_bfloat16 kt = __float2bfloat16_rn(kr), vt = __float2bfloat16_rn(vv[j]);
            if (!a.kv_ready) {
                kc[(int64_t)pos * HD + j] = kt;
                vc[(int64_t)pos * HD + j] = vt;
            }
            kn_s[j] = __bfloat162float(kt);
            vn_s[j] = __bfloat162float(vt);
        }
        __syncthreads();
        uint32_t qa[KS][4];
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            qa[k][0] = pack_bf16(q_s[h * HD + 16 * k + kq], q_s[h * HD + 16 * k + kq + 1]);
            qa[k][1] = 0u;
            qa[k][2] = pack_bf16(q_s[h * HD + 16 * k + 8 + kq], q_s[h * HD + 16 * k + 8 + kq + 1]);
            qa[k][3] = 0u;
        }
        float o[NT][4];
#pragma unroll
        for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
        float m_run = -INFINITY, l_run = 0.f;
        const int n_chunks = pos / CP + 1;
        for (int ci = 0; ci < n_chunks; ++ci, ++seq) {
            const int buf = (int)(seq % NBUF);
            const uint32_t k_s = sbase + buf * kBufBytes, v_s = k_s + CB * kBlockBytes;
            uint8_t* kb = base + buf * kBufBytes;
            const int c0 = ci * CP;
            const int cn = min(CP, pos + 1 - c0);
            if ((int)threadIdx.x < CP) dep_s[threadIdx.x] = dep_reg;
            load_dep();  // the following chunk's depth bytes
            mbar_wait(smem_u32(&bars[buf]), (seq / NBUF) & 1u);
            if (!a.kv_ready && pos < c0 + CP) {  // the new position lives in this chunk: patch it (swizzled)
                const int r = pos - c0;
                for (int j = threadIdx.x; j < HD; j += blockDim.x) {
                    const uint32_t off = (j / 64) * kBlockBytes + swz(r, (j % 64) / 8) + (j % 8) * 2;
                    *reinterpret_cast<__nv_bfloat16*>(kb + off) = __float2bfloat16_rn(kn_s[j]);
                    *reinterpret_cast<__nv_bfloat16*>(kb + CB * kBlockBytes + off) = __float2bfloat16_rn(vn_s[j]);
                }
            }
            __syncthreads();
            const int n_tiles = (cn + 7) / 8;
            float sc[TPW][2];
            int my_tiles = 0;
            float cmax = -INFINITY;
#pragma unroll
            for (int tt = 0; tt < TPW; ++tt) {
                const int t = warp + tt * NW;
                sc[tt][0] = sc[tt][1] = -INFINITY;
                if (t >= n_tiles) continue;
                my_tiles = tt + 1;
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                const int row = t * 8 + (lane & 7);
#pragma unroll
                for (int k2 = 0; k2 < KS; k2 += 2) {
                    const int mi = lane >> 3;
                    const int dim = 16 * (k2 + (mi >> 1)) + 8 * (mi & 1);
                    uint32_t b[4];
                    ldsm_x4(k_s + (dim / 64) * kBlockBytes + swz(row, (dim % 64) / 8), b);
                    mma_bf16(c, qa[k2], b[0], b[1]);
                    mma_bf16(c, qa[k2 + 1], b[2], b[3]);
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int pl = t * 8 + kq + e;
                    const int p = c0 + pl;
                    const bool valid = h < G && p <= pos && (p == pos || dep_s[pl] >= a.layer);
                    sc[tt][e] = valid ? c[e] : -INFINITY;
                    cmax = fmaxf(cmax, sc[tt][e]);
                }
            }
            cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, 1));
            cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, 2));
            const float m_new = fmaxf(m_run, cmax);
            const float scale = m_new == -INFINITY ? 1.f : __expf(m_run - m_new);
            float psum = 0.f;
#pragma unroll
            for (int tt = 0; tt < TPW; ++tt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float p = sc[tt][e] == -INFINITY ? 0.f : __expf(sc[tt][e] - m_new);
                    sc[tt][e] = p;
                    psum += p;
                }
            psum += __shfl_xor_sync(0xffffffffu, psum, 1);
            psum += __shfl_xor_sync(0xffffffffu, psum, 2);
            l_run = l_run * scale + psum;
            m_run = m_new;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                o[n][0] *= scale;
                o[n][1] *= scale;
            }
#pragma unroll
            for (int tt = 0; tt < TPW; tt += 2) {
                if (tt >= my_tiles) break;
                const int ta = warp + tt * NW;
                const bool has_b = tt + 1 < my_tiles;
                const int tb = has_b ? ta + NW : ta;
                uint32_t pa[4];
                pa[0] = pack_bf16(sc[tt][0], sc[tt][1]);
                pa[1] = 0u;
                pa[2] = has_b ? pack_bf16(sc[tt + 1][0], sc[tt + 1][1]) : 0u;
                pa[3] = 0u;
                const int mi = lane >> 3;
                const int row = ((mi & 1) ? tb : ta) * 8 + (lane & 7);
#pragma unroll
                for (int n = 0; n < NT; n += 2) {
                    const int dim = 8 * (n + (mi >> 1));
                    uint32_t b[4];
                    ldsm_x4_t(v_s + (dim / 64) * kBlockBytes + swz(row, (dim % 64) / 8), b);
                    mma_bf16(o[n], pa, b[0], b[1]);
                    mma_bf16(o[n + 1], pa, b[2], b[3]);
                }
            }
            __syncthreads();  // every warp is done reading this buffer
            if (ci + 1 < n_chunks && threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the patch writes
                issue_next(buf);
            }
            if (ci + 1 == n_chunks) {
                // combine the four warps through this (drained) buffer, then refill it
                float* comb = reinterpret_cast<float*>(kb);
                float* ml = comb + NW * 8 * HD;
                if (h < G) {
#pragma unroll
                    for (int n = 0; n < NT; ++n) {
                        comb[(warp * 8 + h) * HD + n * 8 + kq] = o[n][0];
                        comb[(warp * 8 + h) * HD + n * 8 + kq + 1] = o[n][1];
                    }
                    if ((lane & 3) == 0) {
                        ml[(warp * 8 + h) * 2] = m_run;
                        ml[(warp * 8 + h) * 2 + 1] = l_run;
                    }
                }
                __syncthreads();
                __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.out) + (int64_t)i * dq;
                for (int idx = threadIdx.x; idx < G * HD; idx += blockDim.x) {
                    const int hh = idx / HD, j = idx % HD;
                    float M = -INFINITY;
                    for (int w = 0; w < NW; ++w) M = fmaxf(M, ml[(w * 8 + hh) * 2]);
                    float num = 0.f, den = 0.f;
                    for (int w = 0; w < NW; ++w) {
                        const float mw = ml[(w * 8 + hh) * 2];
                        const float f = mw == -INFINITY ? 0.f : __expf(mw - M);
                        num += f * comb[(w * 8 + hh) * HD + j];
                        den += f * ml[(w * 8 + hh) * 2 + 1];
                    }
                    out[(g * G + hh) * HD + j] = __float2bfloat16_rn(num / den);
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    // generic-proxy writes to this buffer precede the async-proxy refill
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue_next(buf);
                }
            }
        }
    }
}

template <int HD>
void launch_pipe(const AttnArgs& a, int num_sms, cudaStream_t s) {
    using C = PipeCfg<HD>;
    const int G = a.n_heads / a.n_kv_heads;
    if (a.splits > 16) throw Error(1, "attention: more than 16 QKV split-K planes");
    const size_t smem = 1024 + PipeSmem<HD>(G, a.splits, a.max_rows).total;
    auto kern = attention_pipe_kernel<HD>;
    EEB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    EEB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NW * 32, smem));
    const int items = a.max_rows * a.n_kv_heads;
    const int grid = std::max(1, std::min(items, std::max(1, per_sm) * num_sms));
    launch_pdl(kern, dim3(grid), dim3(C::NW * 32), smem, s, *static_cast<const CUtensorMap*>(a.k_map),
               *static_cast<const CUtensorMap*>(a.v_map), a);
    EEB_CHECK_LAUNCH();
}

// Fixed-order sum of the QKV GEMM's split-K planes for 4 consecutive columns
// (plane order, as the attention kernels sum them: the same floats result),
// kBatch planes in flight per round trip.
__device__ __forceinline__ float4 plane_sum4(const float* src, int splits, int64_t stride) {
    constexpr int kBatch = 8;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < splits; s0 += kBatch) {
        float4 t[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j)
            if (s0 + j < splits) t[j] = __ldcg(reinterpret_cast<const float4*>(src + (s0 + j) * stride));
#pragma unroll
        for (int j = 0; j < kBatch; ++j)
            if (s0 + j < splits) {
                acc.x += t[j].x;
                acc.y += t[j].y;
                acc.z += t[j].z;
                acc.w += t[j].w;
            }
    }
    return acc;
}
template <typename T>
__device__ __forceinline__ void store4_kv(T* dst, float x, float y, float z, float w) {
    if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(dst) = make_float4(x, y, z, w);
    } else {
        __nv_bfloat162 lo = __floats2bfloat162_rn(x, y), hi = __floats2bfloat162_rn(z, w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(dst) = u;
    }
}

// Prefill: RoPE the keys and append K/V of every live row (one CTA per row;
// a thread owns 4 dims of each half of a key head, or 4 dims of a value head).
template <typename T, bool ONE>
__global__ void kv_append_kernel(Stamp stamp, AttnArgs a) {
    StampScope stamp_scope(stamp);
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.x;
    if (i >= *a.n_active) return;
    const int Hkv = a.n_kv_heads, hd = a.head_dim, half = hd / 2;
    const int dq = a.n_heads * hd, dkv = Hkv * hd;
    const int slot = a.slot[i], pos = a.pos[i];
    const float* row = a.qkv + (int64_t)i * (dq + 2 * dkv);
    const float* cs = a.rope_cos + (int64_t)pos * half;
    const float* sn = a.rope_sin + (int64_t)pos * half;
    T* kc = static_cast<T*>(a.k_cache);
    T* vc = static_cast<T*>(a.v_cache);
    // index idx = (kv head g, 4 dims jj of the first half): the key pair
    // (jj, jj + half) rotated, and the value's same two 4-dim groups — every
    // load of an index in flight before the first use (one round trip)
    const int q4 = half / 4;
    for (int idx = threadIdx.x; idx < Hkv * q4; idx += blockDim.x) {
        const int g = idx / q4, jj = 4 * (idx % q4);
        // (one plane — the cuBLASLt prefill GEMMs — is a plain load: the
        //  8-plane batches of plane_sum4 would hold 32 float4 registers)
        const float* kr = row + dq + g * hd + jj;
        const float* vr = row + dq + dkv + g * hd + jj;
        constexpr bool one = ONE;
        const float4 x0 = one ? __ldcg(reinterpret_cast<const float4*>(kr)) : plane_sum4(kr, a.splits, a.split_stride);
        const float4 x1 = one ? __ldcg(reinterpret_cast<const float4*>(kr + half))
                              : plane_sum4(kr + half, a.splits, a.split_stride);
        const float4 v0 = one ? __ldcg(reinterpret_cast<const float4*>(vr)) : plane_sum4(vr, a.splits, a.split_stride);
        const float4 v1 = one ? __ldcg(reinterpret_cast<const float4*>(vr + half))
                              : plane_sum4(vr + half, a.splits, a.split_stride);
        const float4 c = *reinterpret_cast<const float4*>(cs + jj);
        const float4 sv = *reinterpret_cast<const float4*>(sn + jj);
        T* dst = kc + kv_elem_offset(a, slot, pos, g);
        store4_kv<T>(dst + jj, x0.x * c.x - x1.x * sv.x, x0.y * c.y - x1.y * sv.y, x0.z * c.z - x1.z * sv.z,
                     x0.w * c.w - x1.w * sv.w);
        store4_kv<T>(dst + jj + half, x0.x * sv.x + x1.x * c.x, x0.y * sv.y + x1.y * c.y, x0.z * sv.z + x1.z * c.z,
                     x0.w * sv.w + x1.w * c.w);
        T* vdst = vc + kv_elem_offset(a, slot, pos, g);
        store4_kv<T>(vdst + jj, v0.x, v0.y, v0.z, v0.w);
        store4_kv<T>(vdst + jj + half, v1.x, v1.y, v1.z, v1.w);
    }
}


// ---------------------------------------------------------------------------
// Prefill attention on the tensor cores (flash-attention forward, mma.sync
// m16n8k16 bf16): one CTA per (query block, query head).  A block is <= 64
// consecutive prompt rows of one sequence; each of the 4 warps owns 16 of
// them.  The block's K/V (its sequence's positions [0, last row's position])
// stream once through double-buffered 64-position TMA chunks shared by all
// 64 query rows — the per-row decode kernel would re-read them per row.
// Masking is the decode rule per row: position p is visible to the row at
// position r iff p <= r and (p == r or kv_depth[p] >= layer).
// ---------------------------------------------------------------------------
// HD: the padded head dim (a multiple of 64: the TMA column blocks and the
// shared-memory rows); HR: the model's head dim (80 for OPT-2.7B: the KV maps'
// rows are 80 wide, so the second column block's dims 80..127 arrive as TMA
// out-of-bounds zeros, and q is zero-padded to match).
template <int HD, bool PAGED, int HR = HD>
__global__ void __launch_bounds__(128)
    attention_prefill_kernel(Stamp stamp, const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                             AttnArgs a) {
    StampScope stamp_scope(stamp);
    static_assert(HR <= HD && HR % 16 == 0, "real head dim within the padded one");
    constexpr int CB = HD / 64, CP = 64, NB = 2;
    constexpr int NT = (HR + 15) / 16 * 2, KS = (HR + 31) / 32 * 2;  // n-tiles / k-steps over the real dims
    constexpr uint32_t kBlockBytes = CP * 128, kBufBytes = 2 * CB * kBlockBytes;
    constexpr int kDep = 1024, kMaxPt = PAGED ? 64 : 1;
    pdl_launch_dependents();
    pdl_wait();
    const int item = blockIdx.y;
    if (item >= *a.pf_n_items) return;
    const int4 it = a.pf_items[item];  // {first row, rows, slot, first position}
    const int hq = blockIdx.x;
    const int H = a.n_heads, Hkv = a.n_kv_heads, G = H / Hkv, g = hq / G;
    const int dq = H * HR, dkv = Hkv * HR, half = HR / 2;
    const int r0 = it.x, nrows = it.y, slot = it.z, p0 = it.w;
    const int last = p0 + nrows - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (sbase - raw);
    __nv_bfloat16* q_s = reinterpret_cast<__nv_bfloat16*>(base + NB * kBufBytes);  // [64][HD]
    __shared__ uint8_t dep_s[kDep];
    __shared__ int pt_s[kMaxPt];
    __shared__ __align__(8) uint64_t bars[NB];
    const int PS = PAGED ? a.page_size : a.max_seq;
    if constexpr (PAGED) {
        for (int t = threadIdx.x; t < a.pages_per_seq && t < kMaxPt; t += blockDim.x)
            pt_s[t] = a.page_table[(int64_t)slot * a.pages_per_seq + t];
        __syncthreads();
    }
    auto page_of = [&](int p) { return PAGED ? pt_s[p / PS] : slot; };
    auto row_of = [&](int p) { return PAGED ? p % PS : p; };
    const int n_chunks = last / CP + 1;
    auto issue = [&](int ci) {  // thread 0
        const int c0 = ci * CP, buf = ci % NB;
        const uint32_t k_s = sbase + buf * kBufBytes, v_s = k_s + CB * kBlockBytes;
        const uint32_t bar = smem_u32(&bars[buf]);
        const int n_load = min(CP, last + 1 - c0);
        const int boxes = (n_load + kBoxRows - 1) / kBoxRows;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)boxes * CB * kBoxRows * 128 * 2)
                     : "memory");
        for (int b = 0; b < boxes; ++b) {
            const int p = c0 + b * kBoxRows;
            const int zc = page_of(p) * Hkv + g;
            for (int cb = 0; cb < CB; ++cb) {
                const uint32_t off = cb * kBlockBytes + b * kBoxRows * 128;
                tma_3d(k_s + off, &kmap, bar, cb * 64, row_of(p), zc);
                tma_3d(v_s + off, &vmap, bar, cb * 64, row_of(p), zc);
            }
        }
    };
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&vmap)) : "memory");
        for (int b = 0; b < NB; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[b])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int c = 0; c < NB && c < n_chunks; ++c) issue(c);
    }
    // queries: fixed-order plane sums, RoPE at each row's position, 1/sqrt(hd), bf16
    const float qscale = rsqrtf((float)HR);
    if constexpr (HR < HD)  // the padding dims of q: zeros (K's arrive as zeros too)
        for (int idx = threadIdx.x; idx < 64 * ((HD - HR) / 4); idx += blockDim.x) {
            const int r = idx / ((HD - HR) / 4), jj = HR + 4 * (idx % ((HD - HR) / 4));
            store4_kv<__nv_bfloat16>(q_s + r * HD + jj, 0.f, 0.f, 0.f, 0.f);
        }
    for (int idx = threadIdx.x; idx < 64 * (half / 4); idx += blockDim.x) {
        const int r = idx / (half / 4), jj = 4 * (idx % (half / 4));
        float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
        if (r < nrows) {
            const float* src = a.qkv + (int64_t)(r0 + r) * (dq + 2 * dkv) + hq * HR + jj;
            lo = plane_sum4(src, a.splits, a.split_stride);
            hi = plane_sum4(src + half, a.splits, a.split_stride);
            const int pos = p0 + r;
            const float4 c = *reinterpret_cast<const float4*>(a.rope_cos + (int64_t)pos * half + jj);
            const float4 sv = *reinterpret_cast<const float4*>(a.rope_sin + (int64_t)pos * half + jj);
            const float4 l2 = make_float4((lo.x * c.x - hi.x * sv.x) * qscale, (lo.y * c.y - hi.y * sv.y) * qscale,
                                          (lo.z * c.z - hi.z * sv.z) * qscale, (lo.w * c.w - hi.w * sv.w) * qscale);
            const float4 h2 = make_float4((lo.x * sv.x + hi.x * c.x) * qscale, (lo.y * sv.y + hi.y * c.y) * qscale,
                                          (lo.z * sv.z + hi.z * c.z) * qscale, (lo.w * sv.w + hi.w * c.w) * qscale);
            lo = l2;
            hi = h2;
        }
        store4_kv<__nv_bfloat16>(q_s + r * HD + jj, lo.x, lo.y, lo.z, lo.w);
        store4_kv<__nv_bfloat16>(q_s + r * HD + jj + half, hi.x, hi.y, hi.z, hi.w);
    }
    {
        const uint8_t* dsrc = a.kv_depth + (int64_t)slot * a.max_seq;
        for (int t = threadIdx.x; t < kDep && t <= last; t += blockDim.x) dep_s[t] = dsrc[t];
    }
    __syncthreads();
    // A fragments of this warp's 16 query rows: rows gq and gq + 8
    const int gq = lane >> 2, kq = (lane & 3) * 2;
    const int ra = 16 * warp + gq, rb = ra + 8;
    auto q2 = [&](int r, int d) { return *reinterpret_cast<const uint32_t*>(q_s + r * HD + d); };
    uint32_t qa[KS][4];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
        qa[k][0] = q2(ra, 16 * k + kq);
        qa[k][1] = q2(rb, 16 * k + kq);
        qa[k][2] = q2(ra, 16 * k + 8 + kq);
        qa[k][3] = q2(rb, 16 * k + 8 + kq);
    }
    const int pos_a = p0 + ra, pos_b = p0 + rb;  // rows >= nrows: masked everywhere, never stored
    const bool live_a = ra < nrows, live_b = rb < nrows;
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
    const uint8_t* depth = a.kv_depth + (int64_t)slot * a.max_seq;
    auto visible = [&](int p, int pos, bool live) {
        return live && p <= pos && (p == pos || (p < kDep ? dep_s[p] : depth[p]) >= a.layer);
    };
    // this warp's rows see no position past its last row
    const int warp_last = min(last, p0 + 16 * warp + 15);
    for (int ci = 0; ci < n_chunks; ++ci) {
        const int c0 = ci * CP, buf = ci % NB;
        const uint32_t k_s = sbase + buf * kBufBytes, v_s = k_s + CB * kBlockBytes;
        mbar_wait(smem_u32(&bars[buf]), (uint32_t)((ci / NB) & 1));
        // tiles the TMA wrote (whole 32-row boxes: an even count); rows past
        // them hold stale shared memory, which may not even be finite
        const int loaded = 4 * ((min(CP, last + 1 - c0) + kBoxRows - 1) / kBoxRows);
        if (c0 <= warp_last) {
            float sc[CP / 8][4];
#pragma unroll
            for (int t = 0; t < CP / 8; ++t) {
                sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = -INFINITY;
                if (t >= loaded) continue;
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                const int row = t * 8 + (lane & 7);
#pragma unroll
                for (int k2 = 0; k2 < KS; k2 += 2) {
                    const int mi = lane >> 3;
                    const int dim = 16 * (k2 + (mi >> 1)) + 8 * (mi & 1);
                    uint32_t b[4];
                    ldsm_x4(k_s + (dim / 64) * kBlockBytes + swz(row, (dim % 64) / 8), b);
                    mma_bf16(c, qa[k2], b[0], b[1]);
                    mma_bf16(c, qa[k2 + 1], b[2], b[3]);
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int p = c0 + t * 8 + kq + e;
                    sc[t][e] = visible(p, pos_a, live_a) ? c[e] : -INFINITY;
                    sc[t][2 + e] = visible(p, pos_b, live_b) ? c[2 + e] : -INFINITY;
                }
            }
            float mxa = -INFINITY, mxb = -INFINITY;
#pragma unroll
            for (int t = 0; t < CP / 8; ++t) {
                mxa = fmaxf(mxa, fmaxf(sc[t][0], sc[t][1]));
                mxb = fmaxf(mxb, fmaxf(sc[t][2], sc[t][3]));
            }
            mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 1));
            mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 2));
            mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 1));
            mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 2));
            const float na = fmaxf(m_a, mxa), nb = fmaxf(m_b, mxb);
            const float sa = na == -INFINITY ? 1.f : __expf(m_a - na), sb = nb == -INFINITY ? 1.f : __expf(m_b - nb);
            float psa = 0.f, psb = 0.f;
#pragma unroll
            for (int t = 0; t < CP / 8; ++t) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    sc[t][e] = sc[t][e] == -INFINITY ? 0.f : __expf(sc[t][e] - na);
                    sc[t][2 + e] = sc[t][2 + e] == -INFINITY ? 0.f : __expf(sc[t][2 + e] - nb);
                    psa += sc[t][e];
                    psb += sc[t][2 + e];
                }
            }
            psa += __shfl_xor_sync(0xffffffffu, psa, 1);
            psa += __shfl_xor_sync(0xffffffffu, psa, 2);
            psb += __shfl_xor_sync(0xffffffffu, psb, 1);
            psb += __shfl_xor_sync(0xffffffffu, psb, 2);
            l_a = l_a * sa + psa;
            l_b = l_b * sb + psb;
            m_a = na;
            m_b = nb;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                o[n][0] *= sa;
                o[n][1] *= sa;
                o[n][2] *= sb;
                o[n][3] *= sb;
            }
            // P.V: k = 16 positions = tiles (2j, 2j+1)
#pragma unroll
            for (int tp = 0; tp < CP / 8; tp += 2) {
                if (tp >= loaded) break;
                uint32_t pa[4];
                pa[0] = pack_bf16(sc[tp][0], sc[tp][1]);
                pa[1] = pack_bf16(sc[tp][2], sc[tp][3]);
                pa[2] = pack_bf16(sc[tp + 1][0], sc[tp + 1][1]);
                pa[3] = pack_bf16(sc[tp + 1][2], sc[tp + 1][3]);
                const int mi = lane >> 3;
                const int row = (tp + (mi & 1)) * 8 + (lane & 7);
#pragma unroll
                for (int n = 0; n < NT; n += 2) {
                    const int dim = 8 * (n + (mi >> 1));
                    uint32_t b[4];
                    ldsm_x4_t(v_s + (dim / 64) * kBlockBytes + swz(row, (dim % 64) / 8), b);
                    mma_bf16(o[n], pa, b[0], b[1]);
                    mma_bf16(o[n + 1], pa, b[2], b[3]);
                }
            }
        }
        __syncthreads();  // every warp is past this chunk: its buffer takes chunk ci + NB
        if (threadIdx.x == 0 && ci + NB < n_chunks) issue(ci + NB);
    }
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.out);
    const float ia = l_a > 0.f ? 1.f / l_a : 0.f, ib = l_b > 0.f ? 1.f / l_b : 0.f;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        const int d = 8 * n + kq;
        if (d >= HR) continue;
        if (live_a)
            *reinterpret_cast<uint32_t*>(out + (int64_t)(r0 + ra) * dq + hq * HR + d) = pack_bf16(o[n][0] * ia, o[n][1] * ia);
        if (live_b)
            *reinterpret_cast<uint32_t*>(out + (int64_t)(r0 + rb) * dq + hq * HR + d) = pack_bf16(o[n][2] * ib, o[n][3] * ib);
    }
}

template <int HD, int HR = HD>
void launch_prefill_attn(const AttnArgs& a, cudaStream_t s) {
    const size_t smem = 1024 + 2 * 2 * (size_t)(HD / 64) * 64 * 128 + 64 * HD * 2;
    const bool paged = a.page_size != a.max_seq;
    auto kern = paged ? attention_prefill_kernel<HD, true, HR> : attention_prefill_kernel<HD, false, HR>;
    EEB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(kern, dim3(a.n_heads, a.pf_max_items), dim3(128), smem, s, *static_cast<const CUtensorMap*>(a.k_map),
               *static_cast<const CUtensorMap*>(a.v_map), a);
    EEB_CHECK_LAUNCH();
}

__global__ void mark_depth_kernel(Stamp stamp, int rows, const int* slot, const int* pos,
                                  uint8_t* kv_depth, int max_seq, int depth) {
    StampScope stamp_scope(stamp);
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows) kv_depth[(int64_t)slot[i] * max_seq + pos[i]] = (uint8_t)depth;
}

template <int HD, int CP, int NB, bool PAGED, int W>
void launch_mma_cp_w(const AttnArgs& a, cudaStream_t s) {
    constexpr int CB = HD / 64;
    const int G = a.n_heads / a.n_kv_heads;
    if (a.splits > 16) throw Error(1, "attention: more than 16 QKV split-K planes");
    const size_t smem = 1024 + (size_t)NB * 2 * CB * CP * 128 + (8 + G + 2) * HD * 4;
    auto kern = attention_mma_kernel<HD, CP, NB, PAGED, W>;
    EEB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // x = kv head, y = row: the live rows' CTAs come first in launch order
    dim3 grid(a.n_kv_heads, a.max_rows, a.kv_part && a.kv_ticket ? a.kv_splits : 1);
    launch_pdl(kern, grid, dim3(W * 32), smem, s, *static_cast<const CUtensorMap*>(a.k_map),
               *static_cast<const CUtensorMap*>(a.v_map), a);
    EEB_CHECK_LAUNCH();
}

template <int HD, int CP, int NB, bool PAGED>
void launch_mma_cp_t(const AttnArgs& a, cudaStream_t s) {
    // EEB_ATTN_WARPS=2: 2-warp CTAs (twice the CTAs per SM, half the cross-warp combine)
    static const int env_w = std::getenv("EEB_ATTN_WARPS") ? std::atoi(std::getenv("EEB_ATTN_WARPS")) : 4;
    if (env_w == 2 && CP / 8 / 2 >= 1) launch_mma_cp_w<HD, CP, NB, PAGED, 2>(a, s);
    else launch_mma_cp_w<HD, CP, NB, PAGED, kMmaWarps>(a, s);
}

template <int HD, int CP, int NB>
void launch_mma_cp(const AttnArgs& a, cudaStream_t s) {
    if (a.page_size != a.max_seq) {
        launch_mma_cp_t<HD, CP, NB, true>(a, s);
    } else {
        launch_mma_cp_t<HD, CP, NB, false>(a, s);
    }
}

// Chunk size: the whole context of a (row, kv head) in one chunk keeps one
// TMA round trip per CTA; a smaller chunk fits more CTAs per SM (more loads
// in flight, prologues overlapping other CTAs' loads).  EEB_ATTN_CP overrides.
template <int HD>
void launch_mma(const AttnArgs& a, cudaStream_t s) {
    static const int env_cp = std::getenv("EEB_ATTN_CP") ? std::atoi(std::getenv("EEB_ATTN_CP")) : 0;
    // measured C2 (hd 64, context 128..227), single-buffered: 64 positions 1.56 ms/step, 128 1.61, 256 1.64
    // C2 (same box): 32-position double-buffered chunks 1.458 ms/step, 64 1.468
    const int cp = env_cp > 0 ? env_cp : (HD == 64 ? 32 : 128);
    static const int env_nb = std::getenv("EEB_ATTN_NB") ? std::atoi(std::getenv("EEB_ATTN_NB")) : 0;
    // double-buffered 64-position chunks at 5 CTAs/SM: C2 1.497 vs 1.565 ms/step
    // single-buffered (same box, two orders)
    const int nb = env_nb > 0 ? env_nb : (cp <= 64 ? 2 : 1);
    if (nb >= 4 && cp <= 32) {
        launch_mma_cp<HD, 32, 4>(a, s);
    } else if (nb >= 2) {
        if (cp <= 32) launch_mma_cp<HD, 32, 2>(a, s);
        else if (cp <= 64) launch_mma_cp<HD, 64, 2>(a, s);
        else launch_mma_cp<HD, 128, 2>(a, s);
    } else {
        if (cp <= 32) launch_mma_cp<HD, 32, 1>(a, s);
        else if (cp <= 64) launch_mma_cp<HD, 64, 1>(a, s);
        else if (cp <= 128) launch_mma_cp<HD, 128, 1>(a, s);
        else launch_mma_cp<HD, 256, 1>(a, s);
    }
}

}  // namespace

void launch_kv_append(const AttnArgs& a, cudaStream_t s) {
    // (one plane: the cuBLASLt prefill GEMMs' output; plain loads, few registers)
    if (a.dtype == 0)
        launch_pdl(a.splits == 1 ? kv_append_kernel<float, true> : kv_append_kernel<float, false>, dim3(a.max_rows),
                   dim3(256), 0, s, a);
    else
        launch_pdl(a.splits == 1 ? kv_append_kernel<__nv_bfloat16, true> : kv_append_kernel<__nv_bfloat16, false>,
                   dim3(a.max_rows), dim3(256), 0, s, a);
    EEB_CHECK_LAUNCH();
}

void launch_mark_depth(int rows, const int* slot, const int* pos, uint8_t* kv_depth, int max_seq, int depth,
                       cudaStream_t s) {
    launch_pdl(mark_depth_kernel, dim3((rows + 255) / 256), dim3(256), 0, s, rows, slot, pos, kv_depth, max_seq, depth);
    EEB_CHECK_LAUNCH();
}

void launch_attention(const AttnArgs& a, cudaStream_t s) {
    const bool paged = a.page_size != a.max_seq;
    static const bool no_pf_attn = std::getenv("EEB_PREFILL_ATTN") && std::atoi(std::getenv("EEB_PREFILL_ATTN")) == 0;
    if (a.kv_ready && a.pf_items && !no_pf_attn && a.dtype == 1 && a.k_map && a.v_map &&
        (a.head_dim == 64 || a.head_dim == 80 || a.head_dim == 128)) {
        // (KV depth of positions >= 1024 is read from global memory, not staged)
        if (a.head_dim == 64) launch_prefill_attn<64>(a, s);
        else if (a.head_dim == 80) launch_prefill_attn<128, 80>(a, s);  // OPT-2.7B
        else launch_prefill_attn<128>(a, s);
        return;
    }
    if (launch_attention_dec(a, s)) return;  // streaming decode kernel (attention_dec.cu)
    if (a.dtype == 1 && a.k_map && a.v_map && a.n_heads / a.n_kv_heads <= 8 &&
        (a.head_dim == 64 || a.head_dim == 128)) {
        if (paged) {  // only the one-item kernel walks page tables
            if (a.head_dim == 64) launch_mma<64>(a, s);
            else launch_mma<128>(a, s);
            return;
        }
        // One (row, kv-head) item per CTA for head_dim 64 (MHA, C2: measured
        // faster than the pipelined walk); the pipelined walk for head_dim 128
        // (GQA, C4).  EEB_ATTN=one|pipe overrides (A/B).
        static const char* env = std::getenv("EEB_ATTN");
        const bool one_item = env ? std::string(env) == "one" : a.head_dim == 64;
        if (one_item) {
            if (a.head_dim == 64) launch_mma<64>(a, s);
            else launch_mma<128>(a, s);
        } else {
            if (a.head_dim == 64) launch_pipe<64>(a, a.num_sms, s);
            else launch_pipe<128>(a, a.num_sms, s);
        }
        return;
    }
    const int G = a.n_heads / a.n_kv_heads;
    if (paged) throw Error(3, "attention: the paged KV pool needs a bf16 model with head_dim 64 or 128");
    if (G > kMaxG || a.head_dim > kMaxHd || a.head_dim % 16 != 0 || a.head_dim / 2 > kThreads)
        throw Error(1, "attention: unsupported head geometry");
    const int esz = a.dtype == 0 ? 4 : 2;
    const int C = kChunkBytes / (a.head_dim * esz);
    const int npg = kThreads / (a.head_dim / 2);
    const size_t sc_floats = std::max((size_t)G * C, (size_t)npg * G * a.head_dim);
    const size_t smem = 2 * kChunkBytes + (size_t)G * a.head_dim * 4 + sc_floats * 4;
    // x = kv head, y = row: the live rows' CTAs come first in launch order
    dim3 grid(a.n_kv_heads, a.max_rows);
    if (a.dtype == 0) {
        EEB_CUDA(cudaFuncSetAttribute(attention_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        launch_pdl(attention_kernel<float>, grid, dim3(kThreads), smem, s, a);
    } else {
        EEB_CUDA(cudaFuncSetAttribute(attention_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        launch_pdl(attention_kernel<__nv_bfloat16>, grid, dim3(kThreads), smem, s, a);
    }
    EEB_CHECK_LAUNCH();
}

}  // namespace eeb
