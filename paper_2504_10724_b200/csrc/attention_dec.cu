// attention_dec.cu — streaming flash-decode attention for the bf16 decode step.
//
// One decode step attends n_active rows x Hkv kv-heads = "items" (C2: 64 x 32
// = 2048 items of ~33 KB of K/V each).  Each item is tiny arithmetic (a GEMV
// per head) over a short context, so what bounds it is latency and
// instruction overhead, not FLOPs: splitting one item's positions over the
// warps of a CTA (the one-item kernel) pays a cross-warp combine, named
// barriers and per-8-position softmax bookkeeping in every warp, and leaves
// the K/V stream latency-bound (~30 us per C2 layer in the captured step
// against ~13 us of HBM time; ncu: 34% of DRAM peak, issue slots 43% busy).
//
// Here one CTA per SM, and each compute WARP owns whole items:
//
//   * prologue (all warps, all of the CTA's items at once, overlapping the
//     first K/V loads): q / k / v summed over the QKV split-K planes, RoPE
//     (q scaled by 1/sqrt(hd)), the new position's K/V rounded to bf16 and
//     appended to the cache, the items' KV-depth bytes staged in smem;
//   * each warp streams its items' K/V as 32-position chunks (one TMA box of
//     K and one of V per 64-dim column block) through its own NRW-deep ring
//     of shared-memory stages, issuing the load of chunk j + NRW as soon as
//     chunk j is consumed (lane 0, after __syncwarp) — no producer warp, no
//     cross-warp handshakes;
//   * per chunk: S = Q K^T on mma.sync (rows = the G query heads of the kv
//     head, padded to 16; four 8-position n-tiles), KV-depth / causal mask,
//     one online-softmax rescale per chunk, O += P V with P reused from the
//     score fragments (two n-tiles = one k16 A operand);
//   * at item end the warp normalises O and writes it (bf16) — no combine.
//
// Arithmetic per item is the same as attention_mma_kernel's (q RoPE'd and
// scaled in f32, packed to bf16; scores and the online softmax in f32; P
// packed to bf16 for P.V), and an item's result does not depend on which
// warp or CTA serves it or on the batch (batch invariance).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "kernels.h"
#include "ptx.cuh"

namespace eeb {

namespace {

using namespace ptx;

constexpr int kCP = 32;           // positions per chunk = one TMA box (rows of the KV tensor maps)
constexpr int kMaxItems = 48;     // items per CTA whose prologue data is staged in smem
constexpr int kMaxPages = 64;     // page-table entries per sequence (paged pool)

template <int HD>
struct DecCfg {
    static constexpr int CB = HD / 64;                 // 64-dim column blocks
    static constexpr uint32_t kBlk = kCP * 128;        // one column block of a chunk (4 KB)
    static constexpr uint32_t kStage = 2 * CB * kBlk;  // K + V of one chunk
    static constexpr int NW = HD == 64 ? 8 : 4;        // compute warps (each owns whole items)
    static constexpr int NRW = 3;                      // ring stages per warp
    static constexpr int kThreads = NW * 32;
};

// Shared-memory plan after the rings (host and device agree).
struct DecSmem {
    size_t q_off, kv_off, dep_off, pt_off, rows_off, total;
    int dep_stride;
    __host__ __device__ DecSmem(int HD, int G, int items, int max_seq, bool paged, size_t ring) {
        q_off = ring;                                        // [items][G][HD] f32, RoPE'd and scaled
        kv_off = q_off + (size_t)items * G * HD * 4;         // [items][2][HD] f32 new k (RoPE'd), v; bf16-rounded
        dep_stride = (max_seq + 15) & ~15;
        dep_off = kv_off + (size_t)items * 2 * HD * 4;       // [items][dep_stride] KV depth bytes
        pt_off = (dep_off + (size_t)items * dep_stride + 15) & ~(size_t)15;  // [items][kMaxPages] (paged)
        rows_off = pt_off + (paged ? (size_t)items * kMaxPages * 4 : 0);     // [items] {slot, pos}
        total = rows_off + (size_t)items * 8 + (size_t)items * HD * 4;       // + RoPE cos / sin [items][HD/2] each
    }
};

template <int HD, bool PAGED>
__global__ void __launch_bounds__(DecCfg<HD>::kThreads, 1)
    attention_dec_kernel(Stamp stamp, const __grid_constant__ CUtensorMap kmap,
                         const __grid_constant__ CUtensorMap vmap, AttnArgs a, int items_cap) {
    StampScope stamp_scope(stamp);
    using C = DecCfg<HD>;
    constexpr int CB = C::CB, NW = C::NW, NRW = C::NRW, NT = HD / 8, KS = HD / 16;
    constexpr uint32_t kBlk = C::kBlk, kStage = C::kStage;
    constexpr int kNT = NW * 32;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (sbase - raw);
    __shared__ __align__(8) uint64_t full[NW][NRW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
    if (t < NW * NRW) mbar_init(smem_u32(&full[t / NRW][t % NRW]), 1);
    if (t == 0) {
        prefetch_tmap(&kmap);
        prefetch_tmap(&vmap);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_launch_dependents();
    pdl_wait();
    stamp_waited(stamp);
    const int Hkv = a.n_kv_heads, G = a.n_heads / Hkv;
    const int dq = a.n_heads * HD, dkv = Hkv * HD, half = HD / 2;
    const int n_items = *a.n_active * Hkv;
    const int grid = gridDim.x;
    const int my = (int)blockIdx.x < n_items ? (n_items - 1 - (int)blockIdx.x) / grid + 1 : 0;
    if (my == 0) return;
    const DecSmem L(HD, G, items_cap, a.max_seq, PAGED, (size_t)NW * NRW * kStage);
    float* q_s = reinterpret_cast<float*>(base + L.q_off);
    float* kv_s = reinterpret_cast<float*>(base + L.kv_off);
    uint8_t* dep_s = base + L.dep_off;
    int* pt_s = reinterpret_cast<int*>(base + L.pt_off);
    int2* rows_s = reinterpret_cast<int2*>(base + L.rows_off);
    const int PS = PAGED ? a.page_size : a.max_seq;

    for (int k = t; k < my; k += kNT) {
        const int row = ((int)blockIdx.x + k * grid) / Hkv;
        rows_s[k] = make_int2(a.slot[row], a.pos[row]);
    }
    __syncthreads();  // also publishes the barrier inits
    if constexpr (PAGED) {
        for (int e = t; e < my * kMaxPages; e += kNT) {
            const int k = e / kMaxPages, j = e % kMaxPages;
            if (j < a.pages_per_seq) pt_s[e] = a.page_table[(int64_t)rows_s[k].x * a.pages_per_seq + j];
        }
        __syncthreads();
    }
    auto page_of = [&](int k, int p) { return PAGED ? pt_s[k * kMaxPages + p / PS] : rows_s[k].x; };

    // ---- this warp's chunk stream: items k = warp, warp + NW, ...; chunk c of
    // item k covers positions [32c, 32c + 32) ∩ [0, pos] ------------------------
    const uint32_t ring = sbase + (uint32_t)warp * NRW * kStage;
    int ik = warp, ic = 0;  // next chunk to issue: item index, chunk index
    auto issue_next = [&](int slot_idx) {  // lane 0: the next chunk of the stream into stage slot_idx
        if (ik >= my) return;
        if (a.dbg & 2) {  // timing experiment: no loads (the stage completes empty)
            mbar_arrive(smem_u32(&full[warp][slot_idx]));
            if (++ic > rows_s[ik].y / kCP) {
                ic = 0;
                ik += NW;
            }
            return;
        }
        const int g = ((int)blockIdx.x + ik * grid) % Hkv, pos = rows_s[ik].y;
        const int p = ic * kCP;
        const uint32_t bar = smem_u32(&full[warp][slot_idx]);
        mbar_expect_tx(bar, (uint32_t)CB * kBlk * 2);
        const uint32_t k_st = ring + (uint32_t)slot_idx * kStage, v_st = k_st + CB * kBlk;
        const int zc = page_of(ik, p) * Hkv + g;
        const int r = PAGED ? p % PS : p;
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
            tma_load_3d(k_st + cb * kBlk, &kmap, bar, cb * 64, r, zc);
            tma_load_3d(v_st + cb * kBlk, &vmap, bar, cb * 64, r, zc);
        }
        if (++ic > pos / kCP) {
            ic = 0;
            ik += NW;
        }
    };
    if (lane == 0)
        for (int s = 0; s < NRW; ++s) issue_next(s);

    // ---- prologue (all warps, every item of the CTA) --------------------------
    // Phase A: every global load in flight together — the q/k/v float4s of up
    // to kR elements per thread over all split-K planes, the KV-depth words and
    // the RoPE rows — then one barrier.
    const float* rope_c = a.rope_cos;
    float* cs_s = reinterpret_cast<float*>(base + L.rows_off + (size_t)items_cap * 8);  // [items][half] cos, then sin
    float* sn_s = cs_s + (size_t)items_cap * half;
    if (!(a.dbg & 4)) {  // (timing experiment 4: no prologue)
        const int n4 = (G + 2) * HD / 4, nq4 = G * HD / 4, total = my * n4;
        constexpr int kR = 4;
        for (int e0 = t; e0 < total; e0 += kR * kNT) {
            float4 acc[kR];
            const float* src[kR];
            float* dst[kR];
#pragma unroll
            for (int r = 0; r < kR; ++r) {
                const int e = min(e0 + r * kNT, total - 1);
                const int k = e / n4, v4 = e % n4;
                const int it = (int)blockIdx.x + k * grid, row = it / Hkv, g = it % Hkv;
                const int col = v4 < nq4 ? g * G * HD + 4 * v4
                              : (v4 < nq4 + HD / 4 ? dq + g * HD + 4 * (v4 - nq4)
                                                   : dq + dkv + g * HD + 4 * (v4 - nq4 - HD / 4));
                src[r] = a.qkv + (int64_t)row * (dq + 2 * dkv) + col;
                dst[r] = v4 < nq4 ? q_s + (size_t)k * G * HD + 4 * v4 : kv_s + (size_t)k * 2 * HD + 4 * (v4 - nq4);
                acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int sp = 0; sp < 16; ++sp) {
                if (sp >= a.splits) break;
#pragma unroll
                for (int r = 0; r < kR; ++r) {
                    const float4 x = __ldcg(reinterpret_cast<const float4*>(src[r] + sp * a.split_stride));
                    acc[r].x += x.x; acc[r].y += x.y; acc[r].z += x.z; acc[r].w += x.w;
                }
            }
#pragma unroll
            for (int r = 0; r < kR; ++r)
                if (e0 + r * kNT < total) *reinterpret_cast<float4*>(dst[r]) = acc[r];
        }
        // KV-depth bytes of each item's earlier positions (4-byte words when rows are word-aligned)
        if ((a.max_seq & 3) == 0) {
            const int wstride = L.dep_stride / 4, n_w = my * wstride;
#pragma unroll 4
            for (int e = t; e < n_w; e += kNT) {
                const int k = e / wstride, w = e - k * wstride;
                if (4 * w < rows_s[k].y)
                    reinterpret_cast<uint32_t*>(dep_s)[e] =
                        reinterpret_cast<const uint32_t*>(a.kv_depth + (int64_t)rows_s[k].x * a.max_seq)[w];
            }
        } else {
            const int n_dep = my * L.dep_stride;
#pragma unroll 4
            for (int e = t; e < n_dep; e += kNT) {
                const int k = e / L.dep_stride, p = e - k * L.dep_stride;
                if (p < rows_s[k].y) dep_s[e] = a.kv_depth[(int64_t)rows_s[k].x * a.max_seq + p];
            }
        }
#pragma unroll 4
        for (int e = t; e < my * half; e += kNT) {
            const int k = e / half, jj = e - k * half;
            cs_s[e] = rope_c[(int64_t)rows_s[k].y * half + jj];
            sn_s[e] = a.rope_sin[(int64_t)rows_s[k].y * half + jj];
        }
    }
    __syncthreads();
    // Phase B: RoPE (q scaled by 1/sqrt(hd)), new k / v rounded to bf16, appended.
    if (!(a.dbg & 8)) {  // (timing experiment 8: no RoPE pass)
        const float qscale = rsqrtf((float)HD);
        const int per = (G + 1) * half;  // rotated pairs: G query heads + the key
        for (int e = t; e < my * per; e += kNT) {
            const int k = e / per, hh = (e % per) / half, jj = e % half;
            const float cs = cs_s[k * half + jj], sn = sn_s[k * half + jj];
            float* v = hh < G ? q_s + ((size_t)k * G + hh) * HD : kv_s + (size_t)k * 2 * HD;
            const float x0 = v[jj], x1 = v[jj + half];
            const float r0 = x0 * cs - x1 * sn, r1 = x0 * sn + x1 * cs;
            if (hh < G) {
                v[jj] = r0 * qscale;
                v[jj + half] = r1 * qscale;
            } else {
                const __nv_bfloat16 b0 = __float2bfloat16_rn(r0), b1 = __float2bfloat16_rn(r1);
                v[jj] = __bfloat162float(b0);
                v[jj + half] = __bfloat162float(b1);
                if (!a.kv_ready && !(a.dbg & 16)) {  // append the new key (experiment 16: no append)
                    const int g = ((int)blockIdx.x + k * grid) % Hkv, pos = rows_s[k].y;
                    const int64_t off = (((int64_t)page_of(k, pos) * Hkv + g) * PS + (PAGED ? pos % PS : pos)) * HD;
                    static_cast<__nv_bfloat16*>(a.k_cache)[off + jj] = b0;
                    static_cast<__nv_bfloat16*>(a.k_cache)[off + jj + half] = b1;
                }
            }
        }
        for (int e = t; e < my * HD; e += kNT) {  // v: bf16-rounded and appended
            const int k = e / HD, j = e - k * HD;
            float* v = kv_s + (size_t)k * 2 * HD + HD + j;
            const __nv_bfloat16 b = __float2bfloat16_rn(*v);
            *v = __bfloat162float(b);
            if (!a.kv_ready && !(a.dbg & 16)) {
                const int g = ((int)blockIdx.x + k * grid) % Hkv, pos = rows_s[k].y;
                const int64_t off = (((int64_t)page_of(k, pos) * Hkv + g) * PS + (PAGED ? pos % PS : pos)) * HD;
                static_cast<__nv_bfloat16*>(a.v_cache)[off + j] = b;
            }
        }
    }
    __syncthreads();

    // ---- this warp's items -----------------------------------------------------
    const int h = lane >> 2, kq = (lane & 3) * 2;
    int u = 0;  // chunks consumed by this warp
    for (int k = warp; k < my; k += NW) {
        const int it = (int)blockIdx.x + k * grid, row = it / Hkv, g = it % Hkv;
        const int pos = rows_s[k].y;
        const uint8_t* dep = dep_s + k * L.dep_stride;
        uint32_t qa[KS][4];  // Q as m16n8k16 A fragments: rows = heads (lane / 4), rows 8..15 zero
        const float* qk = q_s + (size_t)k * G * HD;
        const bool hv = h < G;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
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
            const int s = u % NRW;
            const int c0 = c * kCP;
            const uint32_t k_st = ring + (uint32_t)s * kStage, v_st = k_st + CB * kBlk;
            mbar_wait(smem_u32(&full[warp][s]), (uint32_t)((u / NRW) & 1));
            if (pos < c0 + kCP) {  // the new position's row of this chunk: K/V from the prologue
                const int r = pos - c0;
                uint8_t* kb = base + (k_st - sbase);
                for (int j = lane; j < HD; j += 32) {
                    const uint32_t off = (j / 64) * kBlk + swz128(r, (j % 64) / 8) + (j % 8) * 2;
                    *reinterpret_cast<__nv_bfloat16*>(kb + off) = __float2bfloat16_rn(kv_s[(size_t)k * 2 * HD + j]);
                    *reinterpret_cast<__nv_bfloat16*>(kb + CB * kBlk + off) =
                        __float2bfloat16_rn(kv_s[(size_t)k * 2 * HD + HD + j]);
                }
                fence_proxy_async_smem();  // generic writes before the stage's next TMA fill
                __syncwarp();
            }
            // scores of the four 8-position n-tiles (C fragment: row h, positions
            // kq, kq+1).  Every row of the chunk's box is loaded cache data
            // (finite), so all tiles are computed branch-free and masked after.
            float cc[4][4];
#pragma unroll
            for (int ti = 0; ti < 4; ++ti) cc[ti][0] = cc[ti][1] = cc[ti][2] = cc[ti][3] = 0.f;
            if (!(a.dbg & 1)) {
#pragma unroll
                for (int k2 = 0; k2 < KS; k2 += 2) {
                    const int mi = lane >> 3;
                    const int dim = 16 * (k2 + (mi >> 1)) + 8 * (mi & 1);
                    uint32_t b[4][4];
#pragma unroll
                    for (int ti = 0; ti < 4; ++ti)
                        ldsm_x4(k_st + (dim / 64) * kBlk + swz128(ti * 8 + (lane & 7), (dim % 64) / 8), b[ti]);
#pragma unroll
                    for (int ti = 0; ti < 4; ++ti) {
                        mma_m16n8k16(cc[ti], qa[k2], b[ti][0], b[ti][1]);
                        mma_m16n8k16(cc[ti], qa[k2 + 1], b[ti][2], b[ti][3]);
                    }
                }
            }
            float sc[4][2];
            float cmax = -INFINITY;
#pragma unroll
            for (int ti = 0; ti < 4; ++ti) {
                const int p0 = c0 + ti * 8 + kq;  // even: both depth bytes in one aligned 16-bit word
                const uint32_t dd = p0 < pos ? *reinterpret_cast<const uint16_t*>(dep + p0) : 0u;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int p = p0 + e;
                    const bool valid = hv && (p == pos || (p < pos && (int)((dd >> (8 * e)) & 0xffu) >= a.layer));
                    sc[ti][e] = valid ? cc[ti][e] : -INFINITY;
                    cmax = fmaxf(cmax, sc[ti][e]);
                }
            }
            cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, 1));
            cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, 2));
            const float m_new = fmaxf(m_run, cmax);
            const float scale = m_new == -INFINITY ? 1.f : __expf(m_run - m_new);
            float psum = 0.f;
#pragma unroll
            for (int ti = 0; ti < 4; ++ti)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float pr = sc[ti][e] == -INFINITY ? 0.f : __expf(sc[ti][e] - m_new);
                    sc[ti][e] = pr;
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
            // O += P V over the two 16-position halves of the chunk (P = 0 past pos)
            if (!(a.dbg & 1)) {
#pragma unroll
                for (int hp = 0; hp < 2; ++hp) {
                    uint32_t pa[4];
                    pa[0] = pack_bf16x2(sc[2 * hp][0], sc[2 * hp][1]);
                    pa[1] = 0u;
                    pa[2] = pack_bf16x2(sc[2 * hp + 1][0], sc[2 * hp + 1][1]);
                    pa[3] = 0u;
                    const int mi = lane >> 3;
                    const int rrow = (2 * hp + (mi & 1)) * 8 + (lane & 7);
#pragma unroll
                    for (int n = 0; n < NT; n += 2) {
                        const int dim = 8 * (n + (mi >> 1));
                        uint32_t b[4];
                        ldsm_x4_t(v_st + (dim / 64) * kBlk + swz128(rrow, (dim % 64) / 8), b);
                        mma_m16n8k16(o[n], pa, b[0], b[1]);
                        mma_m16n8k16(o[n + 1], pa, b[2], b[3]);
                    }
                }
            }
            __syncwarp();  // every lane is done with the stage
            if (lane == 0) issue_next(s);
        }
        if (hv) {
            __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.out) + (int64_t)row * dq + (g * G + h) * HD;
            const float inv = 1.f / l_run;
#pragma unroll
            for (int n = 0; n < NT; ++n)
                *reinterpret_cast<uint32_t*>(out + n * 8 + kq) = pack_bf16x2(o[n][0] * inv, o[n][1] * inv);
        }
    }
}

template <int HD, bool PAGED>
bool launch_dec(const AttnArgs& a0, cudaStream_t s) {
    using C = DecCfg<HD>;
    AttnArgs a = a0;
    static const int dbg = std::getenv("EEB_ATTN_DBG") ? std::atoi(std::getenv("EEB_ATTN_DBG")) : 0;
    a.dbg = dbg;
    const int G = a.n_heads / a.n_kv_heads;
    const int items_max = a.max_rows * a.n_kv_heads;
    const int grid = std::max(std::min(items_max, a.num_sms), (items_max + kMaxItems - 1) / kMaxItems);
    const int cap = (items_max + grid - 1) / grid;
    const DecSmem L(HD, G, cap, a.max_seq, PAGED, (size_t)C::NW * C::NRW * C::kStage);
    const size_t smem = 1024 + L.total;
    if (smem > 227 * 1024) return false;
    auto kern = attention_dec_kernel<HD, PAGED>;
    EEB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(kern, dim3(grid), dim3(C::kThreads), smem, s, *static_cast<const CUtensorMap*>(a.k_map),
               *static_cast<const CUtensorMap*>(a.v_map), a, cap);
    EEB_CHECK_LAUNCH();
    return true;
}

// ============================================================================
// MHA decode attention on the CUDA cores (one query head per kv head, head_dim
// 64: the OPT shapes of C2 / C3).  With G = 1 an m16n8k16 score tile carries
// one useful row in sixteen, and the per-chunk fragment / online-softmax
// bookkeeping of the kernel above is what bounds it (measured: the kernel
// with its K/V loads and MMAs switched off still takes ~11 us per C2 layer).
// Here each warp owns whole (row, head) items and walks them in two passes
// over its own TMA ring of 32-position chunks:
//
//   K pass  lane = position: the lane's K row (128 B, 128B-swizzled by the
//           TMA, so the 8 lanes of a quarter-warp hit 8 distinct bank groups)
//           dotted with q held in 64 registers; masked scores -> per-warp smem;
//   softmax one warp max and one warp sum per item (no online rescaling);
//   V pass  lane = 2 output dims: every position's V row is one conflict-free
//           128-byte warp load, weighted by the broadcast probabilities.
//
// The item prologue (q / k / v summed over the QKV split-K planes, RoPE, the
// new position's K / V rounded to bf16 and appended to the cache) is per warp
// and overlaps the warp's first chunk loads; there is no CTA-wide barrier.
// Arithmetic is f32 throughout (q is not rounded to bf16; exp via __expf),
// and an item's result does not depend on which warp serves it or on the
// batch.
// ============================================================================
constexpr int kMRows = 32;              // positions per chunk (one TMA box)
constexpr uint32_t kMStage = kMRows * 128;  // one chunk of K or V: 32 rows x 64 bf16
constexpr int kMItems = 8;              // items per warp (host sizes the grid)

struct MhaSmem {
    int ring, s_pad;
    size_t ring_off, sc_off, dep_off, q_off, total;
    __host__ __device__ MhaSmem(int kMW, int nring, int max_seq) {
        ring = nring;
        s_pad = (max_seq + 31) & ~31;
        ring_off = 0;                                                  // [warp][ring] 4 KB stages
        sc_off = (size_t)kMW * nring * kMStage;                        // [warp][s_pad] f32 scores / probabilities
        dep_off = sc_off + (size_t)kMW * s_pad * 4;                    // [warp][s_pad] KV-depth bytes
        q_off = dep_off + (size_t)kMW * s_pad;                         // [warp][2][64] f32 q, new k
        total = q_off + (size_t)kMW * 128 * 4;
    }
};

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <int kMW, bool PAGED>
__global__ void __launch_bounds__(kMW * 32, 1)
    attention_mha_kernel(Stamp stamp, const __grid_constant__ CUtensorMap kmap,
                         const __grid_constant__ CUtensorMap vmap, const __grid_constant__ CUtensorMap kmap8,
                         const __grid_constant__ CUtensorMap vmap8, AttnArgs a, int nring) {
    StampScope stamp_scope(stamp);
    constexpr int HD = 64;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (sbase - raw);
    __shared__ __align__(8) uint64_t full[kMW][4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane < nring) {
        mbar_init(smem_u32(&full[warp][lane]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        prefetch_tmap(&kmap);
        prefetch_tmap(&vmap);
        prefetch_tmap(&kmap8);
        prefetch_tmap(&vmap8);
    }
    __syncwarp();
    pdl_launch_dependents();
    pdl_wait();
    stamp_waited(stamp);
    if (warp == kMW - 1) l2_prefetch_share(a.pf, a.pf_bytes, lane);  // the O GEMM's weights -> L2

    const int H = a.n_heads, S = a.max_seq;
    const int dq = H * HD;
    const int n_items = *a.n_active * H;
    // items of this warp: it = gw, gw + nw, ... (warp-major over the grid so
    // every CTA gets a share of a small batch)
    const int gw = warp * gridDim.x + blockIdx.x, nw = gridDim.x * kMW;
    const int my = gw < n_items ? (n_items - 1 - gw) / nw + 1 : 0;
    if (my == 0) return;
    const MhaSmem L(kMW, nring, S);
    const uint32_t ring = sbase + (uint32_t)(L.ring_off + (size_t)warp * nring * kMStage);
    float* sc_s = reinterpret_cast<float*>(base + L.sc_off) + (size_t)warp * L.s_pad;
    uint8_t* dep_s = base + L.dep_off + (size_t)warp * L.s_pad;
    float* q_s = reinterpret_cast<float*>(base + L.q_off) + warp * 128;
    float* knew_s = q_s + 64;

    // lane k < my holds item k's row, slot, position (shuffled out on demand)
    int i_slot = 0, i_pos = 0;
    if (lane < my) {
        const int row = (gw + lane * nw) / H;
        i_slot = a.slot[row];
        i_pos = a.pos[row];
    }
    // paged: lane j holds page j of the item being issued (and of the next)
    const int PS = PAGED ? a.page_size : S;
    int pg_cur = 0, pg_nxt = 0;
    auto load_pages = [&](int k) {
        const int sl = __shfl_sync(0xffffffffu, i_slot, k & 31);
        return (PAGED && k < my && lane < a.pages_per_seq) ? a.page_table[(int64_t)sl * a.pages_per_seq + lane] : 0;
    };
    if (PAGED) {
        pg_cur = load_pages(0);
        pg_nxt = load_pages(1);
    }

    // ---- the warp's chunk stream: item k, pass ph (0 K, 1 V), chunk ic -------
    int ik = 0, iph = 0, ic = 0;
    auto issue_next = [&](int st) {  // whole warp (shuffles); lane 0 issues
        if (ik >= my) return;
        const int pos = __shfl_sync(0xffffffffu, i_pos, ik);
        const int slot = __shfl_sync(0xffffffffu, i_slot, ik);
        const int g = (gw + ik * nw) % H;
        const int p = ic * kMRows;
        const int page = PAGED ? __shfl_sync(0xffffffffu, pg_cur, p / PS) : slot;
        if (lane == 0) {
            const uint32_t bar = smem_u32(&full[warp][st]), dst = ring + (uint32_t)st * kMStage;
            const int r = PAGED ? p % PS : p, z = page * H + g;
            const int rows = pos + 1 - p;  // positions of this chunk the item attends
            if (rows >= kMRows) {
                mbar_expect_tx(bar, kMStage);
                tma_load_3d(dst, iph == 0 ? &kmap : &vmap, bar, 0, r, z);
            } else {  // the pass's last chunk: 8-row boxes up to pos (one 1 KB swizzle atom each)
                const int n8 = (rows + 7) >> 3;
                mbar_expect_tx(bar, (uint32_t)n8 * 1024u);
                for (int b = 0; b < n8; ++b) tma_load_3d(dst + 1024u * b, iph == 0 ? &kmap8 : &vmap8, bar, 0, r + 8 * b, z);
            }
        }
        if (++ic > pos / kMRows) {
            ic = 0;
            if (++iph == 2) {
                iph = 0;
                ++ik;
                if (PAGED) {
                    pg_cur = pg_nxt;
                    pg_nxt = load_pages(ik + 1);
                }
            }
        }
    };
    for (int st = 0; st < nring; ++st) issue_next(st);

    int u = 0;  // chunks consumed by this warp
    const float qscale = 0.125f;  // 1 / sqrt(64), exact
    for (int k = 0; k < my; ++k) {
        const int it = gw + k * nw, row = it / H, g = it % H;
        const int pos = __shfl_sync(0xffffffffu, i_pos, k);
        const int slot = __shfl_sync(0xffffffffu, i_slot, k);
        // ---- item prologue: lane = dims (2 lane, 2 lane + 1) -----------------
        // every global load of the prologue in flight together: KV-depth words
        // of the item's earlier positions (S % 4 == 0 checked on the host; the
        // first 1024 positions here, the rest below), the RoPE row, the planes
        const uint32_t* dep_g = reinterpret_cast<const uint32_t*>(a.kv_depth + (int64_t)slot * S);
        uint32_t dw[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int w = lane + 32 * i;
            dw[i] = 4 * w < pos ? __ldg(dep_g + w) : 0u;
        }
        // RoPE over pairs (j, j + 32): lane l < 16 holds the first halves, l + 16 the partners
        const int jj = (2 * lane) & 31;
        const float2 cc = __ldg(reinterpret_cast<const float2*>(a.rope_cos + (int64_t)pos * 32 + jj));
        const float2 ss = __ldg(reinterpret_cast<const float2*>(a.rope_sin + (int64_t)pos * 32 + jj));
        const float* src = a.qkv + (int64_t)row * (dq + 2 * dq) + g * HD + 2 * lane;
        float2 q2 = make_float2(0.f, 0.f), k2 = q2, v2 = q2;
#pragma unroll
        for (int sp = 0; sp < 16; ++sp) {
            if (sp >= a.splits) break;
            const float* pl = src + sp * a.split_stride;
            const float2 x = __ldcg(reinterpret_cast<const float2*>(pl));
            const float2 y = __ldcg(reinterpret_cast<const float2*>(pl + dq));
            const float2 z = __ldcg(reinterpret_cast<const float2*>(pl + 2 * dq));
            q2.x += x.x; q2.y += x.y; k2.x += y.x; k2.y += y.y; v2.x += z.x; v2.y += z.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (4 * (lane + 32 * i) < pos) reinterpret_cast<uint32_t*>(dep_s)[lane + 32 * i] = dw[i];
        for (int w = lane + 256; 4 * w < pos; w += 32) reinterpret_cast<uint32_t*>(dep_s)[w] = dep_g[w];
        const float c0 = cc.x, c1 = cc.y, s0 = ss.x, s1 = ss.y;
        const float qp0 = __shfl_xor_sync(0xffffffffu, q2.x, 16), qp1 = __shfl_xor_sync(0xffffffffu, q2.y, 16);
        const float kp0 = __shfl_xor_sync(0xffffffffu, k2.x, 16), kp1 = __shfl_xor_sync(0xffffffffu, k2.y, 16);
        float qr0, qr1, kr0, kr1;
        if (lane < 16) {  // x0 = mine, x1 = partner: x0 cos - x1 sin
            qr0 = q2.x * c0 - qp0 * s0; qr1 = q2.y * c1 - qp1 * s1;
            kr0 = k2.x * c0 - kp0 * s0; kr1 = k2.y * c1 - kp1 * s1;
        } else {          // x1 = mine, x0 = partner: x0 sin + x1 cos
            qr0 = qp0 * s0 + q2.x * c0; qr1 = qp1 * s1 + q2.y * c1;
            kr0 = kp0 * s0 + k2.x * c0; kr1 = kp1 * s1 + k2.y * c1;
        }
        const __nv_bfloat162 kb = __floats2bfloat162_rn(kr0, kr1), vb = __floats2bfloat162_rn(v2.x, v2.y);
        const float vn0 = __low2float(vb), vn1 = __high2float(vb);
        *reinterpret_cast<float2*>(q_s + 2 * lane) = make_float2(qr0 * qscale, qr1 * qscale);
        *reinterpret_cast<float2*>(knew_s + 2 * lane) = make_float2(__low2float(kb), __high2float(kb));
        if (!a.kv_ready) {  // append the new position's K / V (the chunk holding it is patched from registers)
            const int64_t off = (((int64_t)(PAGED ? a.page_table[(int64_t)slot * a.pages_per_seq + pos / PS] : slot) * H +
                                  g) * PS + (PAGED ? pos % PS : pos)) * HD + 2 * lane;
            *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(a.k_cache) + off) = kb;
            *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(a.v_cache) + off) = vb;
        }
        __syncwarp();
        float q[HD];
#pragma unroll
        for (int j = 0; j < HD; j += 4) {
            const float4 t = *reinterpret_cast<const float4*>(q_s + j);
            q[j] = t.x; q[j + 1] = t.y; q[j + 2] = t.z; q[j + 3] = t.w;
        }
        const int nch = pos / kMRows + 1;
        // ---- K pass: lane = position ------------------------------------------
        float mx = -INFINITY;
        for (int c = 0; c < nch; ++c, ++u) {
            const int st = u % nring;
            const uint32_t stage = ring + (uint32_t)st * kMStage;
            mbar_wait(smem_u32(&full[warp][st]), (uint32_t)((u / nring) & 1));
            const int p = c * kMRows + lane;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            if (p != pos) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    uint4 w;
                    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                                 : "r"(stage + swz128(lane, j)));
                    acc[0] = fmaf(q[8 * j + 0], bf_lo(w.x), acc[0]);
                    acc[1] = fmaf(q[8 * j + 1], bf_hi(w.x), acc[1]);
                    acc[2] = fmaf(q[8 * j + 2], bf_lo(w.y), acc[2]);
                    acc[3] = fmaf(q[8 * j + 3], bf_hi(w.y), acc[3]);
                    acc[0] = fmaf(q[8 * j + 4], bf_lo(w.z), acc[0]);
                    acc[1] = fmaf(q[8 * j + 5], bf_hi(w.z), acc[1]);
                    acc[2] = fmaf(q[8 * j + 6], bf_lo(w.w), acc[2]);
                    acc[3] = fmaf(q[8 * j + 7], bf_hi(w.w), acc[3]);
                }
            } else {  // the new position: K from the prologue
#pragma unroll
                for (int j = 0; j < HD; j += 4) {
                    const float4 t = *reinterpret_cast<const float4*>(knew_s + j);
                    acc[0] = fmaf(q[j], t.x, acc[0]);
                    acc[1] = fmaf(q[j + 1], t.y, acc[1]);
                    acc[2] = fmaf(q[j + 2], t.z, acc[2]);
                    acc[3] = fmaf(q[j + 3], t.w, acc[3]);
                }
            }
            const float sc = (acc[0] + acc[1]) + (acc[2] + acc[3]);
            const bool valid = p == pos || (p < pos && (int)dep_s[p] >= a.layer);
            const float s = valid ? sc : -INFINITY;
            if (p <= pos) sc_s[p] = s;
            mx = fmaxf(mx, s);
            __syncwarp();  // every lane is done with the stage
            issue_next(st);
        }
        // ---- softmax over the item's positions (one max, one sum) --------------
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float lsum = 0.f;
        for (int p = lane; p <= pos; p += 32) {
            const float s = sc_s[p];
            const float e = s == -INFINITY ? 0.f : __expf(s - mx);
            sc_s[p] = e;
            lsum += e;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        __syncwarp();
        // ---- V pass: lane = dims (2 lane, 2 lane + 1) -------------------------
        float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
        const uint32_t voff = ((uint32_t)(lane & 3) << 2);
        for (int c = 0; c < nch; ++c, ++u) {
            const int st = u % nring;
            const uint32_t stage = ring + (uint32_t)st * kMStage;
            mbar_wait(smem_u32(&full[warp][st]), (uint32_t)((u / nring) & 1));
            const int c0r = c * kMRows;
            if (c0r + kMRows <= pos) {  // every row precedes the new position
#pragma unroll
                for (int r = 0; r < kMRows; r += 4) {
                    const float4 e = *reinterpret_cast<const float4*>(sc_s + c0r + r);
                    uint32_t w0, w1, w2, w3;
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w0) : "r"(stage + swz128(r, lane >> 2) + voff));
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w1) : "r"(stage + swz128(r + 1, lane >> 2) + voff));
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w2) : "r"(stage + swz128(r + 2, lane >> 2) + voff));
                    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w3) : "r"(stage + swz128(r + 3, lane >> 2) + voff));
                    o0 = fmaf(e.x, bf_lo(w0), o0); o1 = fmaf(e.x, bf_hi(w0), o1);
                    o2 = fmaf(e.y, bf_lo(w1), o2); o3 = fmaf(e.y, bf_hi(w1), o3);
                    o0 = fmaf(e.z, bf_lo(w2), o0); o1 = fmaf(e.z, bf_hi(w2), o1);
                    o2 = fmaf(e.w, bf_lo(w3), o2); o3 = fmaf(e.w, bf_hi(w3), o3);
                }
            } else {  // the item's last chunk: rows up to pos, the new row from registers
                const int nr = pos + 1 - c0r;
                for (int r = 0; r < nr; ++r) {
                    const float e = sc_s[c0r + r];
                    float x0, x1;
                    if (c0r + r == pos) {
                        x0 = vn0;
                        x1 = vn1;
                    } else {
                        uint32_t w;
                        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w) : "r"(stage + swz128(r, lane >> 2) + voff));
                        x0 = bf_lo(w);
                        x1 = bf_hi(w);
                    }
                    o0 = fmaf(e, x0, o0);
                    o1 = fmaf(e, x1, o1);
                }
            }
            __syncwarp();
            issue_next(st);
        }
        const float inv = 1.f / lsum;
        *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(a.out) + (int64_t)row * dq + g * HD + 2 * lane) =
            __floats2bfloat162_rn((o0 + o2) * inv, (o1 + o3) * inv);
    }
}

template <int kMW, bool PAGED>
bool launch_mha_w(const AttnArgs& a, cudaStream_t s) {
    const int items_max = a.max_rows * a.n_kv_heads;
    const int grid = std::max(a.num_sms, (items_max + kMW * kMItems - 1) / (kMW * kMItems));
    if ((items_max + grid * kMW - 1) / (grid * kMW) > std::min(kMItems, 32)) return false;
    int nring = 3;
    while (nring > 2 && 1024 + MhaSmem(kMW, nring, a.max_seq).total > 227 * 1024) --nring;
    const size_t smem = 1024 + MhaSmem(kMW, nring, a.max_seq).total;
    if (smem > 227 * 1024) return false;
    auto kern = attention_mha_kernel<kMW, PAGED>;
    EEB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(kern, dim3(grid), dim3(kMW * 32), smem, s, *static_cast<const CUtensorMap*>(a.k_map),
               *static_cast<const CUtensorMap*>(a.v_map), *static_cast<const CUtensorMap*>(a.k_map8),
               *static_cast<const CUtensorMap*>(a.v_map8), a, nring);
    EEB_CHECK_LAUNCH();
    return true;
}

template <bool PAGED>
bool launch_mha(const AttnArgs& a, cudaStream_t s) {
    static const int warps = std::getenv("EEB_MHA_WARPS") ? std::atoi(std::getenv("EEB_MHA_WARPS")) : 16;
    return warps == 8 ? launch_mha_w<8, PAGED>(a, s) : launch_mha_w<16, PAGED>(a, s);
}

}  // namespace

bool launch_attention_dec(const AttnArgs& a, cudaStream_t s) {
    static const char* env = std::getenv("EEB_ATTN");
    if (env && std::string(env) != "dec" && std::string(env) != "mha") return false;  // A/B against the one-item / pipelined kernels
    static const bool no_mha = env && std::string(env) == "dec";
    if (!no_mha && a.dtype == 1 && !a.kv_ready && a.k_map && a.v_map && a.k_map8 && a.v_map8 && a.splits <= 16 &&
        !a.kv_part &&
        a.n_heads == a.n_kv_heads && a.head_dim == 64 && a.max_seq % 4 == 0) {
        const bool paged = a.page_size != a.max_seq;
        if (!paged || (a.page_size % kMRows == 0 && a.pages_per_seq <= 32))
            if (paged ? launch_mha<true>(a, s) : launch_mha<false>(a, s)) return true;
    }
    if (a.dtype != 1 || a.kv_ready || !a.k_map || !a.v_map || a.splits > 16 || a.kv_part) return false;
    const int G = a.n_heads / a.n_kv_heads;
    if (G > 8 || (a.head_dim != 64 && a.head_dim != 128)) return false;
    const bool paged = a.page_size != a.max_seq;
    if (paged && (a.pages_per_seq > kMaxPages || a.page_size % kCP != 0)) return false;
    if (a.head_dim == 64) return paged ? launch_dec<64, true>(a, s) : launch_dec<64, false>(a, s);
    return paged ? launch_dec<128, true>(a, s) : launch_dec<128, false>(a, s);
}

}  // namespace eeb
