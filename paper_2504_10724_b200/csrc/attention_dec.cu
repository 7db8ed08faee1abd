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
    // + NW helper warps for the prologue (q / k / v plane sums, KV-depth and
    // RoPE staging, RoPE + K/V append) only: twice the loads in flight per
    // round trip (34B B=64: the prologue took 11 of the 20 us per layer)
    static constexpr int NH = NW;
    static constexpr int kThreads = (NW + NH) * 32;
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

// NRW: ring stages per warp (DecCfg's 3; 2 when a large batch's per-CTA
// prologue staging would not fit beside three)
template <int HD, bool PAGED, int NRW>
__global__ void __launch_bounds__(DecCfg<HD>::kThreads, 1)
    attention_dec_kernel(Stamp stamp, const __grid_constant__ CUtensorMap kmap,
                         const __grid_constant__ CUtensorMap vmap, AttnArgs a, int items_cap) {
    StampScope stamp_scope(stamp);
    using C = DecCfg<HD>;
    constexpr int CB = C::CB, NW = C::NW, NT = HD / 8, KS = HD / 16;
    constexpr uint32_t kBlk = C::kBlk, kStage = C::kStage;
    constexpr int kNT = C::kThreads;  // prologue loops: every warp, helpers included
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
    // ring stages issued before the prologue (a.pre_stages; the rest after it)
    const int pre = min(NRW, a.pre_stages);
    if (lane == 0 && warp < NW)
        for (int s = 0; s < pre; ++s) issue_next(s);

    // ---- prologue (all warps, every item of the CTA) --------------------------
    // Phase A: every global load in flight together — the q/k/v float4s of up
    // to kR elements per thread over all split-K planes, the KV-depth words and
    // the RoPE rows — then one barrier.
    const float* rope_c = a.rope_cos;
    float* cs_s = reinterpret_cast<float*>(base + L.rows_off + (size_t)items_cap * 8);  // [items][half] cos, then sin
    float* sn_s = cs_s + (size_t)items_cap * half;
    if (!(a.dbg & 4)) {  // (timing experiment 4: no prologue)
        const int n4 = (G + 2) * HD / 4, nq4 = G * HD / 4, total = my * n4;
        constexpr int kR = 8;
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
    if (t == 0) stamp_mark(stamp);  // (timeline) prologue done
    if (warp >= NW) return;  // helper warps: prologue only
    if (lane == 0)
        for (int s = pre; s < NRW; ++s) issue_next(s);

    // ---- this warp's items -----------------------------------------------------
    const int h = lane >> 2, kq = (lane & 3) * 2;    int u = 0;  // chunks consumed by this warp
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
    static const int env_pre = std::getenv("EEB_ATTN_PRE") ? std::atoi(std::getenv("EEB_ATTN_PRE")) : 1;
    a.pre_stages = env_pre;
    const int G = a.n_heads / a.n_kv_heads;
    const int items_max = a.max_rows * a.n_kv_heads;
    const int grid0 = std::max(std::min(items_max, a.num_sms), (items_max + kMaxItems - 1) / kMaxItems);
    // The CTA stages its items' prologue data (q, new k / v, KV depth, RoPE)
    // beside the warps' rings: at large batch (34B at 256 rows: 2048 items, 14
    // per CTA, 57 KB of q) that does not fit next to 3-deep rings; take 2-deep
    // rings, then more CTAs (fewer items each), before giving up.
    int grid = grid0, nrw = C::NRW;
    size_t smem = 0;
    for (;;) {
        const int cap = (items_max + grid - 1) / grid;
        smem = 1024 + DecSmem(HD, G, cap, a.max_seq, PAGED, (size_t)C::NW * nrw * C::kStage).total;
        if (smem <= 227 * 1024) break;
        if (nrw == C::NRW) {
            nrw = 2;
        } else if (cap > 1) {
            grid += a.num_sms;
        } else {
            return false;
        }
    }
    const int cap = (items_max + grid - 1) / grid;
    auto kern = nrw == 2 ? attention_dec_kernel<HD, PAGED, 2> : attention_dec_kernel<HD, PAGED, C::NRW>;
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
// bookkeeping of the kernel above is what bounds it.  Here each warp owns
// whole (row, head) items and walks each in two passes over its own ring:
//
//   K pass  lane = position: the lane's K row (128 B) dotted with q held in
//           64 registers, read in a lane-rotated 16-byte-chunk order (lane l
//           reads chunk (j + l) mod 8 at step j, with q rotated the same way)
//           so the 8 lanes of a quarter-warp hit 8 distinct bank groups;
//           masked scores -> per-warp smem;
//   softmax one warp max and one warp sum per item (no online rescaling);
//   V pass  lane = 2 output dims: every position's V row is one conflict-free
//           128-byte warp load, weighted by the broadcast probabilities.
//
// K / V move by 1-D bulk copies (cp.async.bulk) of exactly the rows an item
// attends — (slot, head) rows are contiguous in the cache (a page's rows in
// the paged pool) — in chunks of R rows: the CTA's stage pool is split over
// its active warps, so with few live rows (after the exits) a warp's chunks
// are large (up to 256 rows) and few, a whole item in flight in 2 copies per
// pass.  Measured in the C2 step, each TMA tensor op of the 32-row-box
// version cost ~60 cycles of issue per SM and the 10-20 ops per item made
// the stream issue-bound at low batch.
//
// The item prologue (q / k / v summed over the QKV split-K planes, RoPE, the
// new position's K / V rounded to bf16 and appended to the cache) is per warp;
// the rows' slot / position are read in the same round trip as the live-row
// count.  Arithmetic is f32 throughout (q is not rounded to bf16; exp via
// __expf); an item's result does not depend on which warp serves it, on the
// chunk size or on the batch.
// ============================================================================
constexpr int kMItems = 8;       // items per warp at most (host sizes the grid)
constexpr int kMMaxRing = 12;    // stages per warp at most
constexpr int kMRowsCta = 8;     // distinct rows of a CTA's (contiguous) item range at most

struct MhaSmem {
    int s_pad;
    size_t sc_off, q_off, rope_off, dep_off, pt_off, total;
    __host__ __device__ MhaSmem(int HD, int kMW, size_t pool, int max_seq) {
        s_pad = (max_seq + 31) & ~31;
        sc_off = pool;                                      // [warp][s_pad] f32 scores / probabilities
        q_off = sc_off + (size_t)kMW * s_pad * 4;           // [warp][2][HD] f32 q, new k
        rope_off = q_off + (size_t)kMW * 2 * HD * 4;        // [row][HD] f32 cos | sin at the row's position
        dep_off = rope_off + (size_t)kMRowsCta * HD * 4;    // [row][s_pad] KV-depth bytes
        pt_off = dep_off + (size_t)kMRowsCta * s_pad;       // [row][32] pages (paged pool)
        total = pt_off + (size_t)kMRowsCta * 32 * 4;
    }
};

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 w;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "r"(a));
    return w;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t w;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w) : "r"(a));
    return w;
}

// HD: head_dim (64, 80, 128); rows of HD bf16 = NC 16-byte chunks; lane l
// owns the dim pairs p = l + 32 t < HD / 2 (t < PPL) in the prologue and the
// V pass.
template <int HD, int kMW, bool PAGED>
__global__ void __launch_bounds__(kMW * 32, 1)
    attention_mha_kernel(Stamp stamp, AttnArgs a, int pool_kb) {
    StampScope stamp_scope(stamp);
    constexpr int NC = HD / 8, NP = HD / 2, HALF = HD / 2, PPL = (NP + 31) / 32;
    constexpr uint32_t kRow = HD * 2;  // bytes per K / V row
    constexpr int kP = 6;              // QKV planes loaded ahead (C2: all of them)
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (sbase - raw);
    __shared__ __align__(8) uint64_t full[kMW][kMMaxRing];
    __shared__ int s_rows, s_slot[kMRowsCta], s_pos[kMRowsCta];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane < kMMaxRing) {
        mbar_init(smem_u32(&full[warp][lane]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_launch_dependents();
    pdl_wait();
    stamp_waited(stamp);

    const int H = a.n_heads, S = a.max_seq;
    const int dq = H * HD;
    const MhaSmem L(HD, kMW, (size_t)pool_kb << 10, S);
    // The step's small shared arrays (live-row count, the rows' slot /
    // position, RoPE rows, KV-depth rows, page rows) are read once per CTA
    // into smem, not per warp (every warp of the grid would hit the same few
    // L2 lines).
    if (threadIdx.x == 0) s_rows = *a.n_active;
    __syncthreads();
    const int n_items = s_rows * H;
    // contiguous item ranges per CTA: a CTA's items share one or two rows
    const int per = (n_items + (int)gridDim.x - 1) / (int)gridDim.x;
    const int beg = (int)blockIdx.x * per, end = min(beg + per, n_items);
    if (beg >= end) return;
    const int r0 = beg / H, nr = (end - 1) / H - r0 + 1;  // <= kMRowsCta (host)
    // this warp's items: beg + warp + kMW k.  The first item's QKV planes
    // (they depend on the row only) are requested now and summed before the
    // next barrier, overlapping the table loads.
    const bool has = beg + warp < end;
    const int my = has ? (end - beg - warp - 1) / kMW + 1 : 0;
    // the QKV sums of one item: lane's pairs, q / k / v
    auto sum_planes = [&](int it, bool on_item, float2 (&q2)[PPL], float2 (&k2)[PPL], float2 (&v2)[PPL], bool first) {
        const int row = it / H, g = it % H;
        const float* src = a.qkv + (int64_t)row * (3 * dq) + g * HD + 2 * lane;
        float2 xs[PPL][kP], ys[PPL][kP], zs[PPL][kP];
#pragma unroll
        for (int t = 0; t < PPL; ++t)
#pragma unroll
            for (int sp = 0; sp < kP; ++sp) {
                const bool on = on_item && sp < a.splits && lane + 32 * t < NP;
                const float* pl = src + 64 * t + (on ? sp : 0) * a.split_stride;
                xs[t][sp] = on ? __ldcg(reinterpret_cast<const float2*>(pl)) : make_float2(0.f, 0.f);
                ys[t][sp] = on ? __ldcg(reinterpret_cast<const float2*>(pl + dq)) : make_float2(0.f, 0.f);
                zs[t][sp] = on ? __ldcg(reinterpret_cast<const float2*>(pl + 2 * dq)) : make_float2(0.f, 0.f);
            }
        if (first && threadIdx.x < nr) {  // (the rows' tables ride the same round trip)
            s_slot[threadIdx.x] = a.slot[r0 + threadIdx.x];
            s_pos[threadIdx.x] = a.pos[r0 + threadIdx.x];
        }
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
            q2[t] = k2[t] = v2[t] = make_float2(0.f, 0.f);
#pragma unroll
            for (int sp = 0; sp < kP; ++sp) {
                q2[t].x += xs[t][sp].x; q2[t].y += xs[t][sp].y; k2[t].x += ys[t][sp].x; k2[t].y += ys[t][sp].y;
                v2[t].x += zs[t][sp].x; v2[t].y += zs[t][sp].y;
            }
            for (int sp = kP; on_item && sp < a.splits && lane + 32 * t < NP; ++sp) {
                const float* pl = src + 64 * t + sp * a.split_stride;
                const float2 x = __ldcg(reinterpret_cast<const float2*>(pl));
                const float2 y = __ldcg(reinterpret_cast<const float2*>(pl + dq));
                const float2 z = __ldcg(reinterpret_cast<const float2*>(pl + 2 * dq));
                q2[t].x += x.x; q2[t].y += x.y; k2[t].x += y.x; k2[t].y += y.y; v2[t].x += z.x; v2[t].y += z.y;
            }
        }
    };
    float2 q2f[PPL], k2f[PPL], v2f[PPL];
    sum_planes(beg + warp, has, q2f, k2f, v2f, true);
    __syncthreads();
    float* rope_s = reinterpret_cast<float*>(base + L.rope_off);
    uint8_t* depc_s = base + L.dep_off;
    int* pt_s = reinterpret_cast<int*>(base + L.pt_off);
    for (int e = threadIdx.x; e < nr * HD; e += kMW * 32) {
        const int t = e / HD, j = e - t * HD;
        rope_s[e] = (j < HALF ? a.rope_cos : a.rope_sin)[(int64_t)s_pos[t] * HALF + (j < HALF ? j : j - HALF)];
    }
    {
        const int wpr = L.s_pad / 4;  // depth words per row (S % 4 == 0: host)
        for (int e = threadIdx.x; e < nr * wpr; e += kMW * 32) {
            const int t = e / wpr, w = e - t * wpr;
            if (4 * w < s_pos[t])
                reinterpret_cast<uint32_t*>(depc_s)[e] =
                    reinterpret_cast<const uint32_t*>(a.kv_depth + (int64_t)s_slot[t] * S)[w];
        }
    }
    if (PAGED)
        for (int e = threadIdx.x; e < nr * 32; e += kMW * 32)
            if ((e & 31) < a.pages_per_seq) pt_s[e] = a.page_table[(int64_t)s_slot[e >> 5] * a.pages_per_seq + (e & 31)];
    __syncthreads();
    if (!has) return;
    const int active = min(kMW, end - beg);
    // the CTA's stage pool is shared by its active warps: chunk rows R (a
    // multiple of 32, <= 256; <= the page size when paged) with >= 3 stages
    const int per_warp = ((pool_kb << 10) / active) & ~1023;     // bytes (1 KB aligned)
    int R = min(256, (per_warp / (3 * (int)kRow)) & ~31);
    if (PAGED) R = min(R, a.page_size);
    R = max(R, 32);
    const int nring = max(2, min(kMMaxRing, per_warp / (R * (int)kRow)));
    const uint32_t stage_bytes = (uint32_t)R * kRow;
    const uint32_t ring = sbase + (uint32_t)warp * (uint32_t)per_warp;
    float* sc_s = reinterpret_cast<float*>(base + L.sc_off) + (size_t)warp * L.s_pad;
    float* q_s = reinterpret_cast<float*>(base + L.q_off) + warp * 2 * HD;
    float* knew_s = q_s + HD;
    const int PS = PAGED ? a.page_size : S;
    const __nv_bfloat16* kc = static_cast<const __nv_bfloat16*>(a.k_cache);
    const __nv_bfloat16* vc = static_cast<const __nv_bfloat16*>(a.v_cache);
    // (slot, head) row p of the cache, in elements
    auto row_off = [&](int lr, int g, int p) -> int64_t {
        const int page = PAGED ? pt_s[lr * 32 + p / PS] : s_slot[lr];
        return (((int64_t)page * H + g) * PS + (PAGED ? p % PS : p)) * HD;
    };
    const uint64_t pol = policy_evict_first();

    // ---- the warp's chunk stream: item ik, pass iph (0 K, 1 V), chunk rows ip.
    // The issue cursor's item (local row, head, rows attended) is set once per item.
    int ik = 0, iph = 0, ip = 0;
    int c_lr = (beg + warp) / H - r0, c_g = (beg + warp) % H, c_n = s_pos[c_lr] + 1;
    auto issue_next = [&](int st) {  // lane 0
        if (ik >= my) return;
        const uint32_t bar = smem_u32(&full[warp][st]);
        const int rows = min(R, c_n - ip);
        if (a.dbg & 2) {  // timing experiment: no loads (the stage completes empty)
            mbar_arrive(bar);
        } else {
            mbar_expect_tx(bar, (uint32_t)rows * kRow);
            bulk_g2s(ring + (uint32_t)st * stage_bytes, (iph == 0 ? kc : vc) + row_off(c_lr, c_g, ip),
                     (uint32_t)rows * kRow, bar, pol);
        }
        ip += R;
        if (ip >= c_n) {
            ip = 0;
            if (++iph == 2) {
                iph = 0;
                if (++ik < my) {
                    const int it = beg + warp + kMW * ik;
                    c_lr = it / H - r0;
                    c_g = it % H;
                    c_n = s_pos[c_lr] + 1;
                }
            }
        }
    };
    if (lane == 0)
        for (int st = 0; st < nring; ++st) issue_next(st);

    int u = 0;  // chunks consumed by this warp
    const float qscale = rsqrtf((float)HD);
    for (int k = 0; k < my; ++k) {
        const int it = beg + warp + kMW * k, row = it / H, g = it % H, lr = row - r0;
        const int pos = s_pos[lr];
        const uint8_t* dep_s = depc_s + (size_t)lr * L.s_pad;
        // ---- item prologue ------------------------------------------------------
        float2 q2[PPL], k2[PPL], v2[PPL];
        if (k == 0) {
#pragma unroll
            for (int t = 0; t < PPL; ++t) { q2[t] = q2f[t]; k2[t] = k2f[t]; v2[t] = v2f[t]; }
        } else {
            sum_planes(it, true, q2, k2, v2, false);
        }
        // RoPE over pairs (j, j + HD/2) through smem: raw q / k, then rotated
#pragma unroll
        for (int t = 0; t < PPL; ++t)
            if (lane + 32 * t < NP) {
                *reinterpret_cast<float2*>(q_s + 2 * (lane + 32 * t)) = q2[t];
                *reinterpret_cast<float2*>(knew_s + 2 * (lane + 32 * t)) = k2[t];
            }
        __syncwarp();
        float qr0[PPL], qr1[PPL], kr0[PPL], kr1[PPL];
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
            const int d0 = 2 * (lane + 32 * t);
            if (d0 >= HD) continue;
            const bool lo = d0 < HALF;
            const int jj = lo ? d0 : d0 - HALF, pd = lo ? d0 + HALF : d0 - HALF;
            const float2 cc = *reinterpret_cast<const float2*>(rope_s + lr * HD + jj);
            const float2 ss = *reinterpret_cast<const float2*>(rope_s + lr * HD + HALF + jj);
            const float2 qp = *reinterpret_cast<const float2*>(q_s + pd);
            const float2 kp = *reinterpret_cast<const float2*>(knew_s + pd);
            if (lo) {  // x0 = mine, x1 = partner: x0 cos - x1 sin
                qr0[t] = q2[t].x * cc.x - qp.x * ss.x; qr1[t] = q2[t].y * cc.y - qp.y * ss.y;
                kr0[t] = k2[t].x * cc.x - kp.x * ss.x; kr1[t] = k2[t].y * cc.y - kp.y * ss.y;
            } else {   // x1 = mine, x0 = partner: x0 sin + x1 cos
                qr0[t] = qp.x * ss.x + q2[t].x * cc.x; qr1[t] = qp.y * ss.y + q2[t].y * cc.y;
                kr0[t] = kp.x * ss.x + k2[t].x * cc.x; kr1[t] = kp.y * ss.y + k2[t].y * cc.y;
            }
        }
        __syncwarp();
        float vn0[PPL], vn1[PPL];
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
            const int d0 = 2 * (lane + 32 * t);
            if (d0 >= HD) continue;
            const __nv_bfloat162 kb = __floats2bfloat162_rn(kr0[t], kr1[t]), vb = __floats2bfloat162_rn(v2[t].x, v2[t].y);
            vn0[t] = __low2float(vb);
            vn1[t] = __high2float(vb);
            *reinterpret_cast<float2*>(q_s + d0) = make_float2(qr0[t] * qscale, qr1[t] * qscale);
            *reinterpret_cast<float2*>(knew_s + d0) = make_float2(__low2float(kb), __high2float(kb));
            if (!a.kv_ready) {  // append the new position's K / V (its row of the last chunk comes from registers)
                const int64_t off = row_off(lr, g, pos) + d0;
                *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(a.k_cache) + off) = kb;
                *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(a.v_cache) + off) = vb;
            }
        }
        __syncwarp();
        if (k == 0 && lane == 0 && warp == 0) stamp_mark(stamp);  // (timeline) first item's prologue done
        // q rotated per lane: qr[8 j + t] = q[8 ((j + lane) mod NC) + t]
        float qr[HD];
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            const int cj = (j + lane) % NC;
            const float4 t0 = *reinterpret_cast<const float4*>(q_s + 8 * cj);
            const float4 t1 = *reinterpret_cast<const float4*>(q_s + 8 * cj + 4);
            qr[8 * j + 0] = t0.x; qr[8 * j + 1] = t0.y; qr[8 * j + 2] = t0.z; qr[8 * j + 3] = t0.w;
            qr[8 * j + 4] = t1.x; qr[8 * j + 5] = t1.y; qr[8 * j + 6] = t1.z; qr[8 * j + 7] = t1.w;
        }
        const int nch = pos / R + 1;
        // ---- K pass: lane = position ------------------------------------------
        float mx = -INFINITY;
        for (int c = 0; c < nch; ++c, ++u) {
            const int st = u % nring;
            const uint32_t stage = ring + (uint32_t)st * stage_bytes;
            mbar_wait(smem_u32(&full[warp][st]), (uint32_t)((u / nring) & 1));
            const int c0r = c * R, rows = (a.dbg & 1) ? 0 : min(R, pos + 1 - c0r);  // (dbg 1: no compute)
            for (int sb = 0; sb < rows; sb += 32) {
                const int r = sb + lane, p = c0r + r;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                if (p < pos) {
#pragma unroll
                    for (int j = 0; j < NC; ++j) {
                        const uint4 w = lds128(stage + (uint32_t)r * kRow + (uint32_t)(((j + lane) % NC) << 4));
                        acc[0] = fmaf(qr[8 * j + 0], bf_lo(w.x), acc[0]);
                        acc[1] = fmaf(qr[8 * j + 1], bf_hi(w.x), acc[1]);
                        acc[2] = fmaf(qr[8 * j + 2], bf_lo(w.y), acc[2]);
                        acc[3] = fmaf(qr[8 * j + 3], bf_hi(w.y), acc[3]);
                        acc[0] = fmaf(qr[8 * j + 4], bf_lo(w.z), acc[0]);
                        acc[1] = fmaf(qr[8 * j + 5], bf_hi(w.z), acc[1]);
                        acc[2] = fmaf(qr[8 * j + 6], bf_lo(w.w), acc[2]);
                        acc[3] = fmaf(qr[8 * j + 7], bf_hi(w.w), acc[3]);
                    }
                } else if (p == pos) {  // the new position: K from the prologue
#pragma unroll
                    for (int j = 0; j < NC; ++j) {
                        const int cj = (j + lane) % NC;
                        const float4 t0 = *reinterpret_cast<const float4*>(knew_s + 8 * cj);
                        const float4 t1 = *reinterpret_cast<const float4*>(knew_s + 8 * cj + 4);
                        acc[0] = fmaf(qr[8 * j + 0], t0.x, acc[0]);
                        acc[1] = fmaf(qr[8 * j + 1], t0.y, acc[1]);
                        acc[2] = fmaf(qr[8 * j + 2], t0.z, acc[2]);
                        acc[3] = fmaf(qr[8 * j + 3], t0.w, acc[3]);
                        acc[0] = fmaf(qr[8 * j + 4], t1.x, acc[0]);
                        acc[1] = fmaf(qr[8 * j + 5], t1.y, acc[1]);
                        acc[2] = fmaf(qr[8 * j + 6], t1.z, acc[2]);
                        acc[3] = fmaf(qr[8 * j + 7], t1.w, acc[3]);
                    }
                }
                const float sc = (acc[0] + acc[1]) + (acc[2] + acc[3]);
                const bool valid = p == pos || (p < pos && (int)dep_s[p] >= a.layer);
                const float sv = valid ? sc : -INFINITY;
                if (p <= pos) sc_s[p] = sv;
                mx = fmaxf(mx, sv);
            }
            __syncwarp();  // every lane is done with the stage
            if (lane == 0) issue_next(st);
        }
        // ---- softmax over the item's positions (one max, one sum) --------------
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float lsum = 0.f;
        for (int p = lane; p <= pos; p += 32) {
            const float sv = sc_s[p];
            const float e = sv == -INFINITY ? 0.f : __expf(sv - mx);
            sc_s[p] = e;
            lsum += e;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        __syncwarp();
        // ---- V pass: lane = its dim pairs ---------------------------------------
        float o[PPL][4];
#pragma unroll
        for (int t = 0; t < PPL; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
        for (int c = 0; c < nch; ++c, ++u) {
            const int st = u % nring;
            const uint32_t stage = ring + (uint32_t)st * stage_bytes;
            mbar_wait(smem_u32(&full[warp][st]), (uint32_t)((u / nring) & 1));
            const int c0r = c * R;
            const int nfull = (a.dbg & 1) ? 0 : min(R, pos - c0r) & ~3;  // rows before pos, in groups of 4
            for (int r = 0; r < nfull; r += 4) {
                const float4 e = *reinterpret_cast<const float4*>(sc_s + c0r + r);
#pragma unroll
                for (int t = 0; t < PPL; ++t) {
                    if (lane + 32 * t >= NP) continue;
                    const uint32_t vo = (uint32_t)(lane + 32 * t) << 2;
                    const uint32_t w0 = lds32(stage + (uint32_t)r * kRow + vo);
                    const uint32_t w1 = lds32(stage + (uint32_t)(r + 1) * kRow + vo);
                    const uint32_t w2 = lds32(stage + (uint32_t)(r + 2) * kRow + vo);
                    const uint32_t w3 = lds32(stage + (uint32_t)(r + 3) * kRow + vo);
                    o[t][0] = fmaf(e.x, bf_lo(w0), o[t][0]); o[t][1] = fmaf(e.x, bf_hi(w0), o[t][1]);
                    o[t][2] = fmaf(e.y, bf_lo(w1), o[t][2]); o[t][3] = fmaf(e.y, bf_hi(w1), o[t][3]);
                    o[t][0] = fmaf(e.z, bf_lo(w2), o[t][0]); o[t][1] = fmaf(e.z, bf_hi(w2), o[t][1]);
                    o[t][2] = fmaf(e.w, bf_lo(w3), o[t][2]); o[t][3] = fmaf(e.w, bf_hi(w3), o[t][3]);
                }
            }
            const int rows = (a.dbg & 1) ? 0 : min(R, pos + 1 - c0r);
            for (int r = nfull; r < rows; ++r) {  // the rest, the new row from registers
                const float e = sc_s[c0r + r];
#pragma unroll
                for (int t = 0; t < PPL; ++t) {
                    if (lane + 32 * t >= NP) continue;
                    float x0, x1;
                    if (c0r + r == pos) {
                        x0 = vn0[t];
                        x1 = vn1[t];
                    } else {
                        const uint32_t w = lds32(stage + (uint32_t)r * kRow + ((uint32_t)(lane + 32 * t) << 2));
                        x0 = bf_lo(w);
                        x1 = bf_hi(w);
                    }
                    o[t][0] = fmaf(e, x0, o[t][0]);
                    o[t][1] = fmaf(e, x1, o[t][1]);
                }
            }
            __syncwarp();
            if (lane == 0) issue_next(st);
        }
        const float inv = 1.f / lsum;
#pragma unroll
        for (int t = 0; t < PPL; ++t)
            if (lane + 32 * t < NP)
                *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(a.out) + (int64_t)row * dq + g * HD +
                                                    2 * (lane + 32 * t)) =
                    __floats2bfloat162_rn((o[t][0] + o[t][2]) * inv, (o[t][1] + o[t][3]) * inv);
    }
}

template <int HD, int kMW, bool PAGED>
bool launch_mha_w(const AttnArgs& a, cudaStream_t s) {
    const int items_max = a.max_rows * a.n_kv_heads;
    const int grid = std::max(a.num_sms, (items_max + kMW * kMItems - 1) / (kMW * kMItems));
    if ((items_max + grid * kMW - 1) / (grid * kMW) > kMItems) return false;
    // a CTA's contiguous item range spans at most kMRowsCta rows (any live count)
    const int per_max = (items_max + grid - 1) / grid;
    if ((per_max + a.n_kv_heads - 1) / a.n_kv_heads + 1 > kMRowsCta) return false;
    // 227 KB less the static barriers; the stage pool takes what the per-warp
    // buffers leave (at least 2 stages of 32 rows per warp)
    constexpr size_t kBudget = 227 * 1024 - (size_t)kMW * kMMaxRing * 8 - 64;
    const size_t fixed = 1024 + MhaSmem(HD, kMW, 0, a.max_seq).total;
    if (fixed + (size_t)kMW * 2 * 32 * HD * 2 > kBudget) return false;
    const int pool_kb = (int)std::min<size_t>((kBudget - fixed) >> 10, 192);
    const size_t smem = fixed + ((size_t)pool_kb << 10);
    auto kern = attention_mha_kernel<HD, kMW, PAGED>;
    EEB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    static const int dbg = std::getenv("EEB_ATTN_DBG") ? std::atoi(std::getenv("EEB_ATTN_DBG")) : 0;
    AttnArgs ad = a;
    ad.dbg = dbg;  // timing experiments: 1 no compute, 2 no K/V loads
    launch_pdl(kern, dim3(grid), dim3(kMW * 32), smem, s, ad, pool_kb);
    EEB_CHECK_LAUNCH();
    return true;
}

// head_dim 64: 16 warps (q in 64 registers); 80 / 128: 8 warps (more
// registers per thread for the wider q and dim pairs)
template <bool PAGED>
bool launch_mha(const AttnArgs& a, cudaStream_t s) {
    switch (a.head_dim) {
        case 64: return launch_mha_w<64, 16, PAGED>(a, s);
        case 80: return launch_mha_w<80, 8, PAGED>(a, s);
        case 128: return launch_mha_w<128, 8, PAGED>(a, s);
        default: return false;
    }
}

}  // namespace

bool launch_attention_dec(const AttnArgs& a, cudaStream_t s) {
    static const char* env = std::getenv("EEB_ATTN");
    if (env && std::string(env) != "dec" && std::string(env) != "mha") return false;  // A/B against the one-item / pipelined kernels
    static const bool no_mha = env && std::string(env) == "dec";
    if (!no_mha && a.dtype == 1 && !a.kv_ready && a.splits <= 16 && !a.kv_part &&
        a.n_heads == a.n_kv_heads && (a.head_dim == 64 || a.head_dim == 80 || a.head_dim == 128) &&
        a.max_seq % 4 == 0) {
        const bool paged = a.page_size != a.max_seq;
        if (!paged || (a.page_size % 32 == 0 && a.pages_per_seq <= 32))
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
