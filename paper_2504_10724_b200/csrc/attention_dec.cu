// attention_dec.cu — streaming flash-decode attention for the bf16 decode step.
//
// One decode step attends n_active rows x Hkv kv-heads = "items" (C2: 64 x 32
// = 2048 items of ~33 KB of K/V each).  A one-item-per-CTA kernel pays a full
// chain of latencies per item (wait -> slot/pos -> TMA round trips -> compute)
// and only ~5 CTAs fit an SM, so the K/V stream is latency-bound (32 us per
// C2 layer in the captured step against 10 us of HBM time).  Here a grid of
// 2 CTAs per SM walks the items with a grid stride and streams their K/V as
// one continuous sequence of 64-position chunks through an NR-deep TMA ring:
//
//   warp 0 (lane 0)  producer: TMA boxes of K and V for chunk after chunk,
//                    across item boundaries, as soon as a ring stage frees;
//   warps 1..4       prologue for ALL of the CTA's items at once (QKV split-K
//                    plane sums, RoPE, the new position's K/V appended to the
//                    cache, KV-depth bytes), overlapping the first TMA round
//                    trip; then per chunk QK^T / online softmax / PV on
//                    mma.sync (warp w owns position tiles w, w+4 of a chunk),
//                    releasing the stage to the producer; per item the four
//                    warps' partials are combined and written.
//
// Arithmetic per item is the same as attention_mma_kernel's (q RoPE'd and
// scaled in f32, packed to bf16; scores and the online softmax in f32; P
// packed to bf16 for P.V), so results do not depend on the batch or on which
// CTA serves an item (batch invariance).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "kernels.h"
#include "ptx.cuh"

namespace eeb {

namespace {

using namespace ptx;

constexpr int kCP = 64;           // positions per chunk
constexpr int kBox = 32;          // positions per TMA box (rows of the KV tensor maps)
constexpr int kCW = 4;            // compute warps
constexpr int kThreads = (1 + kCW) * 32;
constexpr int kMaxItems = 32;     // items per CTA whose prologue data is staged in smem
constexpr int kMaxPages = 64;     // page-table entries per sequence (paged pool)

template <int HD>
struct DecCfg {
    static constexpr int CB = HD / 64;                 // 64-dim column blocks
    static constexpr uint32_t kBlk = kCP * 128;        // one column block of a chunk
    static constexpr uint32_t kStage = 2 * CB * kBlk;  // K + V of one chunk
    static constexpr int NR = HD == 64 ? 5 : 3;        // ring stages (80 / 96 KB)
};

// Shared-memory plan after the ring (host and device agree).
struct DecSmem {
    size_t q_off, kv_off, dep_off, pt_off, comb_off, ml_off, rows_off, total;
    int dep_stride;
    __host__ __device__ DecSmem(int HD, int G, int items, int max_seq, bool paged, size_t ring) {
        q_off = ring;                                        // [items][G][HD] f32, RoPE'd and scaled
        kv_off = q_off + (size_t)items * G * HD * 4;         // [items][2][HD] f32 new k (RoPE'd), v; bf16-rounded
        dep_stride = (max_seq + 15) & ~15;
        dep_off = kv_off + (size_t)items * 2 * HD * 4;       // [items][dep_stride] KV depth bytes
        pt_off = (dep_off + (size_t)items * dep_stride + 15) & ~(size_t)15;  // [items][kMaxPages] (paged)
        comb_off = pt_off + (paged ? (size_t)items * kMaxPages * 4 : 0);     // [kCW][8][HD] f32
        ml_off = comb_off + (size_t)kCW * 8 * HD * 4;        // [kCW][8][2]
        rows_off = ml_off + (size_t)kCW * 8 * 2 * 4;         // [items] {slot, pos}
        total = rows_off + (size_t)items * 8;
    }
};

template <int HD, bool PAGED>
__global__ void __launch_bounds__(kThreads, 2)
    attention_dec_kernel(Stamp stamp, const __grid_constant__ CUtensorMap kmap,
                         const __grid_constant__ CUtensorMap vmap, AttnArgs a, int items_cap) {
    StampScope stamp_scope(stamp);
    using C = DecCfg<HD>;
    constexpr int CB = C::CB, NR = C::NR, NT = HD / 8, KS = HD / 16, TPW = kCP / 8 / kCW;
    constexpr uint32_t kBlk = C::kBlk, kStage = C::kStage;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (sbase - raw);
    __shared__ __align__(8) uint64_t full[NR], empty[NR];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        prefetch_tmap(&kmap);
        prefetch_tmap(&vmap);
        for (int s = 0; s < NR; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_launch_dependents();
    pdl_wait();
    const int Hkv = a.n_kv_heads, G = a.n_heads / Hkv;
    const int dq = a.n_heads * HD, dkv = Hkv * HD, half = HD / 2;
    const int n_items = *a.n_active * Hkv;
    const int grid = gridDim.x;
    const int my = (int)blockIdx.x < n_items ? (n_items - 1 - (int)blockIdx.x) / grid + 1 : 0;
    if (my == 0) return;
    const DecSmem L(HD, G, items_cap, a.max_seq, PAGED, (size_t)NR * kStage);
    float* q_s = reinterpret_cast<float*>(base + L.q_off);
    float* kv_s = reinterpret_cast<float*>(base + L.kv_off);
    uint8_t* dep_s = base + L.dep_off;
    int* pt_s = reinterpret_cast<int*>(base + L.pt_off);
    float* comb = reinterpret_cast<float*>(base + L.comb_off);
    float* ml = reinterpret_cast<float*>(base + L.ml_off);
    int2* rows_s = reinterpret_cast<int2*>(base + L.rows_off);
    const int PS = PAGED ? a.page_size : a.max_seq;

    for (int k = threadIdx.x; k < my; k += blockDim.x) {
        const int row = ((int)blockIdx.x + k * grid) / Hkv;
        rows_s[k] = make_int2(a.slot[row], a.pos[row]);
    }
    __syncthreads();
    if constexpr (PAGED) {
        for (int e = threadIdx.x; e < my * kMaxPages; e += blockDim.x) {
            const int k = e / kMaxPages, t = e % kMaxPages;
            if (t < a.pages_per_seq) pt_s[e] = a.page_table[(int64_t)rows_s[k].x * a.pages_per_seq + t];
        }
        __syncthreads();
    }
    auto page_of = [&](int k, int p) { return PAGED ? pt_s[k * kMaxPages + p / PS] : rows_s[k].x; };

    if (warp == 0) {
        // ---- producer: chunk after chunk through the ring ----------------------
        if (lane == 0) {
            int u = 0;  // ring use counter
            for (int k = 0; k < my; ++k) {
                const int g = ((int)blockIdx.x + k * grid) % Hkv, pos = rows_s[k].y;
                const int nch = pos / kCP + 1;
                for (int c = 0; c < nch; ++c, ++u) {
                    const int s = u % NR;
                    mbar_wait(smem_u32(&empty[s]), (uint32_t)(((u / NR) & 1) ^ 1));
                    const int c0 = c * kCP;
                    // boxes covering [c0, pos] (the box holding pos too: every
                    // row a score tile touches is finite cache data)
                    const int boxes = (min(kCP, pos + 1 - c0) + kBox - 1) / kBox;
                    const uint32_t bar = smem_u32(&full[s]);
                    mbar_expect_tx(bar, (uint32_t)boxes * CB * kBox * 128 * 2);
                    const uint32_t k_st = sbase + (uint32_t)s * kStage, v_st = k_st + CB * kBlk;
                    for (int b = 0; b < boxes; ++b) {
                        const int p = c0 + b * kBox;
                        const int zc = page_of(k, p) * Hkv + g;
                        const int r = PAGED ? p % PS : p;
#pragma unroll
                        for (int cb = 0; cb < CB; ++cb) {
                            const uint32_t off = cb * kBlk + b * kBox * 128;
                            tma_load_3d(k_st + off, &kmap, bar, cb * 64, r, zc);
                            tma_load_3d(v_st + off, &vmap, bar, cb * 64, r, zc);
                        }
                    }
                }
            }
        }
        return;
    }

    // ---- compute warps ----------------------------------------------------------
    const int t = threadIdx.x - 32, cw = warp - 1;
    constexpr int kNT = kCW * 32;
    // prologue, pass 1: q / k / v of every item summed over the QKV split-K planes
    {
        const int n4 = (G + 2) * HD / 4, nq4 = G * HD / 4;
        for (int e = t; e < my * n4; e += kNT) {
            const int k = e / n4, v4 = e % n4;
            const int it = (int)blockIdx.x + k * grid, row = it / Hkv, g = it % Hkv;
            const int col = v4 < nq4 ? g * G * HD + 4 * v4
                          : (v4 < nq4 + HD / 4 ? dq + g * HD + 4 * (v4 - nq4) : dq + dkv + g * HD + 4 * (v4 - nq4 - HD / 4));
            const float* src = a.qkv + (int64_t)row * (dq + 2 * dkv) + col;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int sp = 0; sp < 16; ++sp) {
                if (sp < a.splits) {
                    const float4 x = *reinterpret_cast<const float4*>(src + sp * a.split_stride);
                    acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
                }
            }
            float* dst = v4 < nq4 ? q_s + (size_t)k * G * HD + 4 * v4 : kv_s + (size_t)k * 2 * HD + 4 * (v4 - nq4);
            *reinterpret_cast<float4*>(dst) = acc;
        }
        // KV depth bytes of every item's earlier positions
        for (int k = 0; k < my; ++k) {
            const int slot = rows_s[k].x, pos = rows_s[k].y;
            const uint8_t* dsrc = a.kv_depth + (int64_t)slot * a.max_seq;
            for (int p = t; p < pos; p += kNT) dep_s[k * L.dep_stride + p] = dsrc[p];
        }
    }
    named_sync(1, kNT);
    // pass 2: RoPE (q scaled by 1/sqrt(hd)), the new K/V rounded to bf16 and appended
    {
        const float qscale = rsqrtf((float)HD);
        const int per = (G + 1) * half;  // rotated pairs: G query heads + the key
        for (int e = t; e < my * per; e += kNT) {
            const int k = e / per, hh = (e % per) / half, jj = e % half;
            const int pos = rows_s[k].y;
            const float cs = a.rope_cos[(int64_t)pos * half + jj], sn = a.rope_sin[(int64_t)pos * half + jj];
            float* v = hh < G ? q_s + ((size_t)k * G + hh) * HD : kv_s + (size_t)k * 2 * HD;
            const float x0 = v[jj], x1 = v[jj + half];
            const float r0 = x0 * cs - x1 * sn, r1 = x0 * sn + x1 * cs;
            if (hh < G) {
                v[jj] = r0 * qscale;
                v[jj + half] = r1 * qscale;
            } else {
                v[jj] = __bfloat162float(__float2bfloat16_rn(r0));
                v[jj + half] = __bfloat162float(__float2bfloat16_rn(r1));
            }
        }
        for (int e = t; e < my * HD; e += kNT) {  // v: bf16-rounded
            const int k = e / HD, j = e % HD;
            float* v = kv_s + (size_t)k * 2 * HD + HD;
            v[j] = __bfloat162float(__float2bfloat16_rn(v[j]));
        }
    }
    named_sync(1, kNT);
    if (!a.kv_ready) {
        for (int e = t; e < my * HD; e += kNT) {
            const int k = e / HD, j = e % HD;
            const int g = ((int)blockIdx.x + k * grid) % Hkv, pos = rows_s[k].y;
            const int64_t off = (((int64_t)page_of(k, pos) * Hkv + g) * PS + (PAGED ? pos % PS : pos)) * HD + j;
            static_cast<__nv_bfloat16*>(a.k_cache)[off] = __float2bfloat16_rn(kv_s[(size_t)k * 2 * HD + j]);
            static_cast<__nv_bfloat16*>(a.v_cache)[off] = __float2bfloat16_rn(kv_s[(size_t)k * 2 * HD + HD + j]);
        }
    }

    const int h = lane >> 2, kq = (lane & 3) * 2;
    int u = 0;
    for (int k = 0; k < my; ++k) {
        const int it = (int)blockIdx.x + k * grid, row = it / Hkv, g = it % Hkv;
        const int pos = rows_s[k].y;
        const uint8_t* dep = dep_s + k * L.dep_stride;
        // Q as m16n8k16 A fragments: rows = heads (lane / 4), rows 8..15 zero
        uint32_t qa[KS][4];
        const float* qk = q_s + (size_t)k * G * HD;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const bool hv = h < G;
            qa[ks][0] = hv ? pack_bf16x2(qk[h * HD + 16 * ks + kq], qk[h * HD + 16 * ks + kq + 1]) : 0u;
            qa[ks][1] = 0u;
            qa[ks][2] = hv ? pack_bf16x2(qk[h * HD + 16 * ks + 8 + kq], qk[h * HD + 16 * ks + 8 + kq + 1]) : 0u;
            qa[ks][3] = 0u;
        }
        float o[NT][4];
#pragma unroll
        for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
        float m_run = -INFINITY, l_run = 0.f;
        const int nch = pos / kCP + 1;
        for (int c = 0; c < nch; ++c, ++u) {
            const int s = u % NR;
            const int c0 = c * kCP, cn = min(kCP, pos + 1 - c0);
            const uint32_t k_st = sbase + (uint32_t)s * kStage, v_st = k_st + CB * kBlk;
            mbar_wait(smem_u32(&full[s]), (uint32_t)((u / NR) & 1));
            if (pos < c0 + kCP) {  // the new position's row of this chunk: K/V from the prologue
                const int r = pos - c0;
                uint8_t* kb = base + (size_t)s * kStage;
                for (int j = t; j < HD; j += kNT) {
                    const uint32_t off = (j / 64) * kBlk + swz128(r, (j % 64) / 8) + (j % 8) * 2;
                    *reinterpret_cast<__nv_bfloat16*>(kb + off) = __float2bfloat16_rn(kv_s[(size_t)k * 2 * HD + j]);
                    *reinterpret_cast<__nv_bfloat16*>(kb + CB * kBlk + off) =
                        __float2bfloat16_rn(kv_s[(size_t)k * 2 * HD + HD + j]);
                }
                fence_proxy_async_smem();  // generic writes before the stage's next TMA fill
                named_sync(1, kNT);
            }
            const int n_tiles = (cn + 7) / 8;
            float sc[TPW][2];
            int my_tiles = 0;
            float cmax = -INFINITY;
#pragma unroll
            for (int tt = 0; tt < TPW; ++tt) {
                const int ti = cw + tt * kCW;
                sc[tt][0] = sc[tt][1] = -INFINITY;
                if (ti >= n_tiles) continue;
                my_tiles = tt + 1;
                float cc[4] = {0.f, 0.f, 0.f, 0.f};
                const int rrow = ti * 8 + (lane & 7);
#pragma unroll
                for (int k2 = 0; k2 < KS; k2 += 2) {
                    const int mi = lane >> 3;
                    const int dim = 16 * (k2 + (mi >> 1)) + 8 * (mi & 1);
                    uint32_t b[4];
                    ldsm_x4(k_st + (dim / 64) * kBlk + swz128(rrow, (dim % 64) / 8), b);
                    mma_m16n8k16(cc, qa[k2], b[0], b[1]);
                    mma_m16n8k16(cc, qa[k2 + 1], b[2], b[3]);
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int p = c0 + ti * 8 + kq + e;
                    const bool valid = h < G && p <= pos && (p == pos || dep[p] >= a.layer);
                    sc[tt][e] = valid ? cc[e] : -INFINITY;
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
                    const float pr = sc[tt][e] == -INFINITY ? 0.f : __expf(sc[tt][e] - m_new);
                    sc[tt][e] = pr;
                    psum += pr;
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
                const int ta = cw + tt * kCW;
                const bool has_b = tt + 1 < my_tiles;
                const int tb = has_b ? ta + kCW : ta;  // pad with a loaded tile, P = 0
                uint32_t pa[4];
                pa[0] = pack_bf16x2(sc[tt][0], sc[tt][1]);
                pa[1] = 0u;
                pa[2] = has_b ? pack_bf16x2(sc[tt + 1][0], sc[tt + 1][1]) : 0u;
                pa[3] = 0u;
                const int mi = lane >> 3;
                const int rrow = ((mi & 1) ? tb : ta) * 8 + (lane & 7);
#pragma unroll
                for (int n = 0; n < NT; n += 2) {
                    const int dim = 8 * (n + (mi >> 1));
                    uint32_t b[4];
                    ldsm_x4_t(v_st + (dim / 64) * kBlk + swz128(rrow, (dim % 64) / 8), b);
                    mma_m16n8k16(o[n], pa, b[0], b[1]);
                    mma_m16n8k16(o[n + 1], pa, b[2], b[3]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&empty[s]));  // this warp is done with the stage
        }
        // combine the compute warps: O = sum_w e^(m_w - M) O_w / sum_w e^(m_w - M) l_w
        if (h < G) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                comb[(cw * 8 + h) * HD + n * 8 + kq] = o[n][0];
                comb[(cw * 8 + h) * HD + n * 8 + kq + 1] = o[n][1];
            }
            if ((lane & 3) == 0) {
                ml[(cw * 8 + h) * 2] = m_run;
                ml[(cw * 8 + h) * 2 + 1] = l_run;
            }
        }
        named_sync(1, kNT);
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.out) + (int64_t)row * dq;
        for (int e = t; e < G * HD; e += kNT) {
            const int hh = e / HD, j = e % HD;
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < kCW; ++w) M = fmaxf(M, ml[(w * 8 + hh) * 2]);
            float num = 0.f, den = 0.f;
#pragma unroll
            for (int w = 0; w < kCW; ++w) {
                const float mw = ml[(w * 8 + hh) * 2];
                const float f = mw == -INFINITY ? 0.f : __expf(mw - M);
                num += f * comb[(w * 8 + hh) * HD + j];
                den += f * ml[(w * 8 + hh) * 2 + 1];
            }
            out[(g * G + hh) * HD + j] = __float2bfloat16_rn(num / den);
        }
        named_sync(1, kNT);  // comb / ml are reused by the next item
    }
}

template <int HD, bool PAGED>
bool launch_dec(const AttnArgs& a, cudaStream_t s) {
    using C = DecCfg<HD>;
    const int G = a.n_heads / a.n_kv_heads;
    const int items_max = a.max_rows * a.n_kv_heads;
    const int grid = std::max(std::min(items_max, 2 * a.num_sms), (items_max + kMaxItems - 1) / kMaxItems);
    const int cap = (items_max + grid - 1) / grid;
    const DecSmem L(HD, G, cap, a.max_seq, PAGED, (size_t)C::NR * C::kStage);
    const size_t smem = 1024 + L.total;
    if (smem > 227 * 1024) return false;
    auto kern = attention_dec_kernel<HD, PAGED>;
    EEB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(kern, dim3(grid), dim3(kThreads), smem, s, *static_cast<const CUtensorMap*>(a.k_map),
               *static_cast<const CUtensorMap*>(a.v_map), a, cap);
    EEB_CHECK_LAUNCH();
    return true;
}

}  // namespace

bool launch_attention_dec(const AttnArgs& a, cudaStream_t s) {
    static const char* env = std::getenv("EEB_ATTN");
    if (env && std::string(env) != "dec") return false;  // A/B against the one-item / pipelined kernels
    if (a.dtype != 1 || a.kv_ready || !a.k_map || !a.v_map || a.splits > 16 || a.kv_part) return false;
    const int G = a.n_heads / a.n_kv_heads;
    if (G > 8 || a.head_dim != 64) return false;
    const bool paged = a.page_size != a.max_seq;
    if (paged && (a.pages_per_seq > kMaxPages || a.page_size % kBox != 0)) return false;
    return paged ? launch_dec<64, true>(a, s) : launch_dec<64, false>(a, s);
}

}  // namespace eeb
