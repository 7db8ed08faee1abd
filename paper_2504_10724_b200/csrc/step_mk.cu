// step_mk.cu — the persistent decode-step kernel (one CTA per SM).
//
// Warp roles (256 threads):
//   warp 0      W producer: walks every GEMM phase of the program and streams
//               this CTA's weight tiles [128 x 64] into the W ring by TMA.  It
//               never waits for a grid barrier — only for ring slots — so the
//               weight stream of phase p+1 overlaps phase p's tail, the
//               barrier and any non-GEMM phase in between;
//   warp 1      TMEM owner + tcgen05.mma issuer (whole warp runs the loop, one
//               elected lane issues; swap-AB: the weight tile is the M=128
//               operand, the batch rows are N); accumulators double-buffered;
//   warp 2      control: grid barriers; X (activation) producer of a GEMM
//               phase — only after the barrier, the activations being the
//               previous phase's output; survivor compaction in DECIDE;
//   warps 2-7   SIMT work of the non-GEMM phases (RMSNorm, attention, MLP
//               activation, exit-head reduction, decision, finalize);
//   warps 4-7   GEMM epilogue: tcgen05.ld (thread = output feature) -> the
//               CTA's partial-sum slots.
// GEMM work is split stream-K: a phase's tiles x k-blocks are cut into G
// equal contiguous ranges, one per CTA, so every SM streams the same number of
// weight bytes.  Consumers reduce the partials of a tile in CTA order (= k
// order): deterministic, no atomics on any value that feeds a logit.
//
// Reference semantics of the decision phases (/root/reference/proj/include/eeserve):
//   confidence = max softmax prob, logprob = log p(argmax) — SPEC.md:106, trace.hpp:17-22;
//   argmax ties -> lowest token id;
//   introspective: first head with confidence >= th exits, final head forced — trace.hpp:69-76;
//   flat: head at / deepest below the serving depth, exit_layer = depth — trace.hpp:86-97, engine.hpp:350-354;
//   breached = conf < th (never at full depth) — engine.hpp:353,358,363; unchanged — engine.hpp:366;
//   histogram = ExitHistogram::add per exit head — pht.hpp:19-22.
#include "../../include/eeb/eeb.h"
#include "kernels.h"
#include "ptx.cuh"
#include "step_mk.cuh"

namespace eeb {
namespace mk {

namespace {

using namespace ptx;

constexpr uint32_t kWStageBytes = kBM * kBK * 2;  // 16 KB
constexpr int kSimtThreads = kSimtWarps * 32;     // 192

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// trace stamps: 0 barrier passed, 1 last X load issued, 2 epilogue done, 3 phase done (before barrier),
// 4 W first issue, 5 W last issue, 6 MMA first k-block, 7 MMA last k-block
constexpr int kStamps = 8;
__device__ __forceinline__ void stamp(const Params& p, int pi, int k) {
    if (p.trace) p.trace[((size_t)blockIdx.x * p.n_phases + pi) * kStamps + k] = gtime();
}

// Stream-K range of CTA c: the first min(G, total) CTAs split the phase's
// k-blocks evenly (so contributing CTAs are consecutive), the rest idle.
__device__ __forceinline__ void cta_range(const Phase& ph, int c, int G, int& s, int& e) {
    const int Gp = min(G, ph.total);
    if (c >= Gp) {
        s = e = ph.total;
        return;
    }
    s = (int)(((long long)ph.total * c) / Gp);
    e = (int)(((long long)ph.total * (c + 1)) / Gp);
}

// Sum over the stream-K segments of GEMM phase `src` for compact row i and NV
// consecutive output columns starting at col (NV-aligned, inside one tile):
// CTA order = k order (deterministic).  All segment loads are issued before
// the in-order sum, so a consumer thread has up to kSegUnroll L2 requests in
// flight.  segtab[t] = {first CTA, its partial slot, segment count}
// (host-computed; Phase::pad[0] = the phase's table offset).
template <int NV>
struct VecF;
template <> struct VecF<1> { using T = float; };
template <> struct VecF<2> { using T = float2; };
template <> struct VecF<4> { using T = float4; };
__device__ __forceinline__ void vadd(float& a, float b) { a += b; }
__device__ __forceinline__ void vadd(float2& a, float2 b) { a.x += b.x; a.y += b.y; }
__device__ __forceinline__ void vadd(float4& a, float4 b) { a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w; }

template <int NV>
__device__ __forceinline__ typename VecF<NV>::T psum(const Params& p, const int4* __restrict__ segtab, const Phase& src,
                                                     int i, int col) {
    using T = typename VecF<NV>::T;
    const int4 sg = segtab[src.pad[0] + (col >> 7)];  // shared memory
    const float* base = p.partials + (size_t)i * kBM + (col & 127);
    const size_t ss = (size_t)p.bpad * kBM;
    T v[kSegUnroll];
#pragma unroll
    for (int j = 0; j < kSegUnroll; ++j)
        if (j < sg.z)
            v[j] = __ldcg(reinterpret_cast<const T*>(base + (size_t)(j == 0 ? sg.x * kMaxSeg + sg.y : (sg.x + j) * kMaxSeg) * ss));
    T acc = v[0];
#pragma unroll
    for (int j = 1; j < kSegUnroll; ++j)
        if (j < sg.z) vadd(acc, v[j]);
    for (int j = kSegUnroll; j < sg.z; ++j)
        vadd(acc, __ldcg(reinterpret_cast<const T*>(base + (size_t)((sg.x + j) * kMaxSeg) * ss)));
    return acc;
}

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }

// Sum over the 192 SIMT threads (warps 2..7), fixed tree (deterministic).
__device__ __forceinline__ float simt_sum(float v, float* red) {
    v = warp_sum(v);
    const int w = (threadIdx.x >> 5) - 2, lane = threadIdx.x & 31;
    if (lane == 0) red[w] = v;
    named_sync(3, kSimtThreads);
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < kSimtWarps; ++k) t += red[k];
    named_sync(3, kSimtThreads);
    return t;
}

// ---------------------------------------------------------------------------
// SIMT phases
// ---------------------------------------------------------------------------
// One CTA per live row; warp w owns 128-column tiles w, w+6, ...; lane = 4
// columns (float4).  The row stays in registers between the two passes.
constexpr int kNormTilesPerWarp = 3;  // D <= 6 * 3 * 128 = 2304 (host-checked)
__device__ __noinline__ void phase_norm(const Params& p, const int4* segtab, const Phase* prog, const Phase& ph,
                                        const int* live, int n_live, float* red) {
    const int w = (threadIdx.x >> 5) - 2, lane = threadIdx.x & 31;
    const float* g = p.gains[ph.gain];
    __nv_bfloat16* out = (ph.flags & kFlagOutHead) ? p.hh : p.h;
    const bool embed = ph.flags & kFlagEmbed;
    if (p.dbg & 64) return;  // timing experiment: empty norm phases
    const bool has_src = ph.src >= 0 && !(p.dbg & 128);  // timing experiment: no partial reads
    const Phase src = ph.src >= 0 ? prog[ph.src] : ph;
    const int tiles = p.D / 128;
    for (int i = blockIdx.x; i < n_live; i += gridDim.x) {
        const int r = live[i];
        float* xr = p.x + (size_t)r * p.D;
        const __nv_bfloat16* er = p.emb + (size_t)p.tok[r] * p.D;
        float4 v[kNormTilesPerWarp], gg[kNormTilesPerWarp];
        // 1) every load of the row slice (and the gains) in flight before any use
#pragma unroll
        for (int k = 0; k < kNormTilesPerWarp; ++k) {
            const int t = w + k * kSimtWarps;
            if (t < tiles) {
                const int c = t * 128 + lane * 4;
                gg[k] = __ldg(reinterpret_cast<const float4*>(g + c));
                if (embed) {
                    const uint2 u = *reinterpret_cast<const uint2*>(er + c);
                    v[k] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                                       __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
                } else {
                    v[k] = __ldcg(reinterpret_cast<const float4*>(xr + c));
                }
            }
        }
        if (has_src) {
#pragma unroll
            for (int k = 0; k < kNormTilesPerWarp; ++k) {
                const int t = w + k * kSimtWarps;
                if (t < tiles) vadd(v[k], psum<4>(p, segtab, src, i, t * 128 + lane * 4));
            }
        }
        // 2) residual write-back and the row's sum of squares
        float ss = 0.f;
#pragma unroll
        for (int k = 0; k < kNormTilesPerWarp; ++k) {
            const int t = w + k * kSimtWarps;
            if (t < tiles) {
                if (embed || has_src) __stcg(reinterpret_cast<float4*>(xr + t * 128 + lane * 4), v[k]);
                ss += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
            }
        }
        ss = simt_sum(ss, red);
        const float inv = rsqrtf(ss / (float)p.D + p.eps);
#pragma unroll
        for (int k = 0; k < kNormTilesPerWarp; ++k) {
            const int t = w + k * kSimtWarps;
            if (t < tiles) {
                const int c = t * 128 + lane * 4;
                const __nv_bfloat162 o0 = __floats2bfloat162_rn(v[k].x * inv * gg[k].x, v[k].y * inv * gg[k].y);
                const __nv_bfloat162 o1 = __floats2bfloat162_rn(v[k].z * inv * gg[k].z, v[k].w * inv * gg[k].w);
                uint2 u;
                u.x = *reinterpret_cast<const uint32_t*>(&o0);
                u.y = *reinterpret_cast<const uint32_t*>(&o1);
                *reinterpret_cast<uint2*>(out + (size_t)i * p.D + c) = u;
            }
        }
    }
}

// Task = (live row, 128-column tile of the up projection); lane = 4 columns.
__device__ __forceinline__ void act_store(const Params& p, bool swiglu, int i, int c, float4 a) {
    if (swiglu) {  // interleaved (gate, up) pairs -> outputs c/2, c/2+1
        const __nv_bfloat162 o = __floats2bfloat162_rn(a.x / (1.f + __expf(-a.x)) * a.y,
                                                      a.z / (1.f + __expf(-a.z)) * a.w);
        *reinterpret_cast<__nv_bfloat162*>(p.hmid + (size_t)i * p.F + c / 2) = o;
    } else {
        const __nv_bfloat162 o0 = __floats2bfloat162_rn(fmaxf(a.x, 0.f), fmaxf(a.y, 0.f));
        const __nv_bfloat162 o1 = __floats2bfloat162_rn(fmaxf(a.z, 0.f), fmaxf(a.w, 0.f));
        uint2 u;
        u.x = *reinterpret_cast<const uint32_t*>(&o0);
        u.y = *reinterpret_cast<const uint32_t*>(&o1);
        *reinterpret_cast<uint2*>(p.hmid + (size_t)i * p.F + c) = u;
    }
}

// Task = (live row, 128-column tile of the up projection); lane = 4 columns;
// two tasks per iteration so both tiles' partial loads are in flight together.
__device__ __noinline__ void phase_act(const Params& p, const int4* segtab, const Phase& src, int n_live) {
    const int w = (threadIdx.x >> 5) - 2, lane = threadIdx.x & 31;
    const int tiles = src.tiles;
    const int ntask = n_live * tiles;
    const bool swiglu = p.mlp_kind == EEB_MLP_SWIGLU;
    const int stride = gridDim.x * kSimtWarps;
    for (int task = blockIdx.x * kSimtWarps + w; task < ntask; task += 2 * stride) {
        const int task2 = task + stride;
        const int i = task / tiles, t = task % tiles;
        const int i2 = task2 / tiles, t2 = task2 % tiles;
        const float4 a = psum<4>(p, segtab, src, i, t * 128 + lane * 4);
        float4 a2 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (task2 < ntask) a2 = psum<4>(p, segtab, src, i2, t2 * 128 + lane * 4);
        act_store(p, swiglu, i, t * 128 + lane * 4, a);
        if (task2 < ntask) act_store(p, swiglu, i2, t2 * 128 + lane * 4, a2);
    }
}

constexpr int kAttnSlots = 4;                                    // (bulk-copy attention variant: see git history)
constexpr int kAttnWarpBytes = 2048 + 512 + kAttnSlots * 4096;
constexpr int kAttnCtlBytes = kAttnSlots * 8 + 8;

// Attention, one warp per (compact row, KV head) task; head_dim 64 (2 dims per
// lane).  Scores: lanes over positions; P.V: lanes over positions with a
// 64-wide accumulator, then a register butterfly leaves dims (2l, 2l+1) in
// lane l.  Masking: a position whose token exited before this layer has no
// K/V here (kv_depth < layer); the current position is always valid.
__device__ __noinline__ void phase_attn(const Params& p, const int4* segtab, const Phase& src, int layer,
                                        const int* live, int n_live, float* scratch, uint8_t* attn_ctl) {
    (void)attn_ctl;
    const int warp = (threadIdx.x >> 5) - 2, lane = threadIdx.x & 31;
    const int Gq = p.H / p.Hkv;
    float* q_s = scratch + warp * (8 * 64 + 128);  // [Gq][64]
    float* kn_s = q_s + 8 * 64;                    // [64] new key (rotated)
    float* vn_s = kn_s + 64;                       // [64] new value
    const float inv_sqrt = rsqrtf(64.f);
    const int d0 = 2 * lane;
    const int ri = lane < 16 ? d0 : d0 - 32;       // rotate-half table index of this lane's dims
    const int ntask = n_live * p.Hkv;
    __nv_bfloat16* kc = p.k_cache + (size_t)(layer - 1) * p.kv_layer_elems;
    __nv_bfloat16* vc = p.v_cache + (size_t)(layer - 1) * p.kv_layer_elems;
    for (int task = blockIdx.x * kSimtWarps + warp; task < ntask; task += gridDim.x * kSimtWarps) {
        const int i = task / p.Hkv, g = task % p.Hkv;
        const int r = live[i];
        const int slot = p.slot[r], pos = p.pos[r];
        const float* cs = p.rope_cos + (size_t)pos * 32;
        const float* sn = p.rope_sin + (size_t)pos * 32;
        const float c0 = cs[ri], c1 = cs[ri + 1], s0 = sn[ri], s1 = sn[ri + 1];
        auto rope = [&](float2 a, float* dst) {
            const float b0 = __shfl_xor_sync(0xffffffffu, a.x, 16), b1 = __shfl_xor_sync(0xffffffffu, a.y, 16);
            if (lane < 16) {
                dst[d0] = a.x * c0 - b0 * s0;
                dst[d0 + 1] = a.y * c1 - b1 * s1;
            } else {
                dst[d0] = b0 * s0 + a.x * c0;
                dst[d0 + 1] = b1 * s1 + a.y * c1;
            }
        };
        for (int hq = 0; hq < Gq; ++hq) rope(psum<2>(p, segtab, src, i, (g * Gq + hq) * 64 + d0), q_s + hq * 64);
        {
            rope(psum<2>(p, segtab, src, i, p.dq + g * 64 + d0), kn_s);
            const float2 v = psum<2>(p, segtab, src, i, p.dq + p.dkv + g * 64 + d0);
            // the cache holds bf16: attend to the rounded values, as later steps will
            const __nv_bfloat162 kb = __floats2bfloat162_rn(kn_s[d0], kn_s[d0 + 1]);
            const __nv_bfloat162 vb = __floats2bfloat162_rn(v.x, v.y);
            kn_s[d0] = __low2float(kb);
            kn_s[d0 + 1] = __high2float(kb);
            vn_s[d0] = __low2float(vb);
            vn_s[d0 + 1] = __high2float(vb);
            const size_t off = (((size_t)slot * p.Hkv + g) * p.S + pos) * 64 + d0;
            *reinterpret_cast<__nv_bfloat162*>(kc + off) = kb;
            *reinterpret_cast<__nv_bfloat162*>(vc + off) = vb;
        }
        __syncwarp();
        const __nv_bfloat16* kbase = kc + ((size_t)slot * p.Hkv + g) * p.S * 64;
        const __nv_bfloat16* vbase = vc + ((size_t)slot * p.Hkv + g) * p.S * 64;
        const uint8_t* dep = p.kv_depth + (size_t)slot * p.S;
        const int npos = pos + 1;
        for (int hq = 0; hq < Gq; ++hq) {
            const float* q = q_s + hq * 64;
            float sc[8];
            float m = -INFINITY;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int pp = lane + 32 * j;
                sc[j] = -INFINITY;
                if (pp < npos && (pp == pos || dep[pp] >= layer)) {
                    float s = 0.f;
                    if (pp == pos) {
#pragma unroll 16
                        for (int d = 0; d < 64; ++d) s += q[d] * kn_s[d];
                    } else {
                        const uint4* kr = reinterpret_cast<const uint4*>(kbase + (size_t)pp * 64);
#pragma unroll
                        for (int v = 0; v < 8; ++v) {
                            const uint4 u = __ldg(kr + v);
                            float f[8];
                            unpack16(u, f, (const __nv_bfloat16*)nullptr);
#pragma unroll
                            for (int e = 0; e < 8; ++e) s += q[v * 8 + e] * f[e];
                        }
                    }
                    sc[j] = s * inv_sqrt;
                    m = fmaxf(m, sc[j]);
                }
            }
            m = warp_max(m);
            float l = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                sc[j] = sc[j] == -INFINITY ? 0.f : __expf(sc[j] - m);
                l += sc[j];
            }
            l = warp_sum(l);
            float acc[64];
#pragma unroll
            for (int d = 0; d < 64; ++d) acc[d] = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int pp = lane + 32 * j;
                if (sc[j] != 0.f) {
                    if (pp == pos) {
#pragma unroll
                        for (int d = 0; d < 64; ++d) acc[d] += sc[j] * vn_s[d];
                    } else {
                        const uint4* vr = reinterpret_cast<const uint4*>(vbase + (size_t)pp * 64);
#pragma unroll
                        for (int v = 0; v < 8; ++v) {
                            const uint4 u = __ldg(vr + v);
                            float f[8];
                            unpack16(u, f, (const __nv_bfloat16*)nullptr);
#pragma unroll
                            for (int e = 0; e < 8; ++e) acc[v * 8 + e] += sc[j] * f[e];
                        }
                    }
                }
            }
            // butterfly: after 5 halvings lane l holds dims (2l, 2l+1)
#pragma unroll
            for (int step = 0; step < 5; ++step) {
                const int o = 16 >> step;
                const int half = 32 >> step;
                const bool upper = lane & o;
#pragma unroll
                for (int d = 0; d < 32; ++d) {
                    if (d < half) {
                        const float send = upper ? acc[d] : acc[d + half];
                        const float keep = upper ? acc[d + half] : acc[d];
                        acc[d] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                    }
                }
            }
            const float invl = 1.f / l;
            const int h = g * Gq + hq;
            *reinterpret_cast<__nv_bfloat162*>(p.attn + (size_t)i * p.dq + h * 64 + d0) =
                __floats2bfloat162_rn(acc[0] * invl, acc[1] * invl);
        }
        __syncwarp();
    }
}

// Online (max, sum-exp, argmax) merge; ties -> lowest token id.
__device__ __forceinline__ void lse_merge(float& m, float& s, int& a, float m2, float s2, int a2) {
    const float M = fmaxf(m, m2);
    const float t1 = m == -INFINITY ? 0.f : s * __expf(m - M);
    const float t2 = m2 == -INFINITY ? 0.f : s2 * __expf(m2 - M);
    a = (m2 > m || (m2 == m && a2 < a)) ? a2 : a;
    s = t1 + t2;
    m = M;
}

// Exit-head reduction, task = (live row, chunk of kHeadChunk vocabulary
// tiles): per-chunk (max, sum-exp, argmax) -> stats[row][chunk]; DECIDE merges
// the chunks in order.  Lane = 4 vocabulary entries per tile.
__device__ __noinline__ void phase_head_reduce(const Params& p, const int4* segtab, const Phase& src, int n_live) {
    const int w = (threadIdx.x >> 5) - 2, lane = threadIdx.x & 31;
    const int nchunk = (src.tiles + kHeadChunk - 1) / kHeadChunk;
    const int ntask = n_live * nchunk;
    for (int task = blockIdx.x * kSimtWarps + w; task < ntask; task += gridDim.x * kSimtWarps) {
        const int i = task / nchunk, ch = task % nchunk;
        float m = -INFINITY, s = 0.f;
        int am = 0x7fffffff;
        const int t1 = min(src.tiles, (ch + 1) * kHeadChunk);
        for (int t = ch * kHeadChunk; t < t1; t += 4) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (t + u < t1) v[u] = psum<4>(p, segtab, src, i, (t + u) * 128 + lane * 4);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (t + u < t1) {
                    const int c = (t + u) * 128 + lane * 4;
                    const float vv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (c + k < p.V) lse_merge(m, s, am, vv[k], 1.f, c + k);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
            const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
            const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
            lse_merge(m, s, am, m2, s2, a2);
        }
        if (lane == 0) p.stats[(size_t)i * nchunk + ch] = make_float4(m, s, __int_as_float(am), 0.f);
    }
}

__device__ __forceinline__ void write_row(const StepOutDev& o, int r, int exit_layer, int tok, float conf,
                                          float logp, int breached, int unchanged, int bin) {
    o.exit_layer[r] = exit_layer;
    o.token_id[r] = tok;
    o.confidence[r] = conf;
    o.logprob[r] = logp;
    o.breached[r] = (uint8_t)breached;
    o.unchanged[r] = (uint8_t)unchanged;
    o.bin[r] = bin;
}

// Warp 2 of every CTA: identical decisions and compaction; CTA 0 writes.
// All SIMT threads: thread i merges row i's vocabulary chunks (in order) into
// {token, confidence, logprob} in shared memory.
__device__ __noinline__ void decide_merge(const Params& p, int nchunk, int n_live, float4* merged) {
    const int t = threadIdx.x - 64;
    for (int i = t; i < n_live; i += kSimtThreads) {
        float m = -INFINITY, S = 0.f;
        int tok = 0x7fffffff;
        for (int c0 = 0; c0 < nchunk; c0 += 16) {
            float4 st[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (c0 + u < nchunk) st[u] = __ldcg(p.stats + (size_t)i * nchunk + c0 + u);
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (c0 + u < nchunk) lse_merge(m, S, tok, st[u].x, st[u].y, __float_as_int(st[u].z));
        }
        merged[i] = make_float4(__int_as_float(tok), 1.f / S, -logf(S), 0.f);
    }
}

__device__ __noinline__ void phase_decide(const Params& p, const Phase& ph, const float4* merged, int* live,
                                          int* n_live_s) {
    const int lane = threadIdx.x & 31;
    const int e = ph.exit_index;
    const bool final = ph.flags & kFlagFinal;
    const bool writer = blockIdx.x == 0;
    const StepOutDev& o = p.out;
    const int n_live = *n_live_s;
    int kept = 0;
    for (int base = 0; base < n_live; base += 32) {
        const int i = base + lane;
        const bool valid = i < n_live;
        int r = 0;
        bool survive = false;
        if (valid) {
            r = live[i];
            const float4 mr = merged[i];
            const int tok = __float_as_int(mr.x);
            const float conf = mr.y, logp = mr.z;
            switch (p.policy) {
                case EEB_FLAT:
                    if (writer)
                        write_row(o, r, p.serving_depth, tok, conf, logp, conf < p.th,
                                  final && ph.exit_layer == p.L ? 1 : 2, e);
                    break;
                case EEB_FULL_DEPTH:
                    if (writer) write_row(o, r, p.L, tok, conf, logp, 0, 1, e);
                    break;
                case EEB_INTROSPECTIVE:
                    if (final) {
                        if (writer) write_row(o, r, ph.exit_layer, tok, conf, logp, conf < p.th, 1, e);
                    } else if (conf >= p.th) {
                        if (writer) write_row(o, r, ph.exit_layer, tok, conf, logp, 0, 2, e);
                    } else {
                        survive = true;
                    }
                    break;
                default:  // EEB_PROFILE
                    if (writer) {
                        const int64_t q0 = (int64_t)r * p.n_exits;
                        o.head_token[q0 + e] = tok;
                        o.head_confidence[q0 + e] = conf;
                        o.head_logprob[q0 + e] = logp;
                        if (final) {
                            int ex = p.n_exits - 1;
                            for (int k = 0; k < p.n_exits; ++k)
                                if (o.head_confidence[q0 + k] >= p.th) { ex = k; break; }
                            write_row(o, r, p.exit_layers[ex], o.head_token[q0 + ex], o.head_confidence[q0 + ex],
                                      o.head_logprob[q0 + ex], o.head_confidence[q0 + ex] < p.th,
                                      o.head_token[q0 + ex] == tok ? 1 : 0, ex);
                        }
                    }
                    break;
            }
        }
        if (p.policy == EEB_INTROSPECTIVE && !final) {
            const unsigned ballot = __ballot_sync(0xffffffffu, survive);
            __syncwarp();
            if (survive) live[kept + __popc(ballot & ((1u << lane) - 1u))] = r;
            kept += __popc(ballot);
            __syncwarp();
        }
    }
    if (p.policy == EEB_INTROSPECTIVE && !final && lane == 0) *n_live_s = kept;
    __syncwarp();
}

__device__ __noinline__ void phase_finalize(const Params& p, float* red) {
    if (blockIdx.x != 0) return;
    const int t = threadIdx.x - 64;
    unsigned* hist_s = reinterpret_cast<unsigned*>(red);  // [64]
    unsigned* breach_s = hist_s + 64;
    for (int k = t; k < 65; k += kSimtThreads) hist_s[k] = 0;
    named_sync(3, kSimtThreads);
    const StepOutDev& o = p.out;
    unsigned my_breach = 0;
    for (int r = t; r < p.batch; r += kSimtThreads) {
        const int b = o.bin[r];
        if (b >= 0 && b < p.n_exits) atomicAdd(hist_s + b, 1u);
        my_breach += o.breached[r] ? 1u : 0u;
        p.kv_depth[(size_t)p.slot[r] * p.S + p.pos[r]] =
            (uint8_t)(p.policy == EEB_PROFILE ? p.L : o.exit_layer[r]);
    }
    atomicAdd(breach_s, my_breach);
    named_sync(3, kSimtThreads);
    if (t < p.n_exits) o.hist[t] = (int64_t)hist_s[t];
    if (t == 0) {
        *o.n_breached = *breach_s;
        double s = 0.0;  // fixed row order
        for (int r = 0; r < p.batch; ++r) s += (double)o.logprob[r];
        *o.sum_logprob = s;
    }
}

struct Smem {
    uint32_t w, x;    // ring bases (shared addresses)
    uint32_t xstage;  // bytes per X stage
    uint32_t wfull, wempty, xfull, xempty, accfull, accempty;  // barrier arrays (8 B apart)
};

__global__ void __launch_bounds__(kThreads, 1) step_kernel(const __grid_constant__ Params p, const int4* segtab_g) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* base_ptr = smem_raw + (base - raw);
    auto ptr_of = [&](uint32_t a) { return base_ptr + (a - base); };
    const int Sw = p.w_stages, Sx = p.x_stages;
    Smem sm;
    sm.xstage = (uint32_t)p.bpad * kBK * 2;
    sm.w = base;
    sm.x = base + (uint32_t)Sw * kWStageBytes;
    const uint32_t bar0 = sm.x + (uint32_t)Sx * sm.xstage;
    sm.wfull = bar0;
    sm.wempty = sm.wfull + 8 * Sw;
    sm.xfull = sm.wempty + 8 * Sw;
    sm.xempty = sm.xfull + 8 * Sx;
    sm.accfull = sm.xempty + 8 * Sx;
    sm.accempty = sm.accfull + 16;
    const uint32_t misc = sm.accempty + 16 + 32;  // 8 B aligned
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ptr_of(misc));
    volatile uint32_t* w_progress = tmem_slot + 1;
    volatile uint32_t* epi_count = tmem_slot + 2;
    int* n_live_s = reinterpret_cast<int*>(tmem_slot + 3);
    float* red = reinterpret_cast<float*>(ptr_of(misc + 64));                // [64 + 1]
    Phase* prog = reinterpret_cast<Phase*>(ptr_of(misc + 64 + 64 * 4 + 64));  // [n_phases]
    int* live = reinterpret_cast<int*>(prog + p.n_phases);                   // [kMaxRows]
    int4* seg_s = reinterpret_cast<int4*>(                                   // [n_segtab], 16 B aligned
        (reinterpret_cast<uintptr_t>(live + kMaxRows) + 15) & ~(uintptr_t)15);
    float* scratch = reinterpret_cast<float*>(ptr_of(sm.x));                 // X ring, idle in SIMT phases

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, blk = blockIdx.x;
    for (int i = threadIdx.x; i < p.n_phases * (int)(sizeof(Phase) / 4); i += blockDim.x)
        reinterpret_cast<int*>(prog)[i] = reinterpret_cast<const int*>(p.phases)[i];
    for (int i = threadIdx.x; i < p.batch; i += blockDim.x) live[i] = i;
    for (int i = threadIdx.x; i < p.n_segtab; i += blockDim.x) seg_s[i] = segtab_g[i];
    const int4* segtab = seg_s;
    uint8_t* attn_ctl = reinterpret_cast<uint8_t*>(seg_s + p.n_segtab);  // [kSimtWarps][kAttnCtlBytes], 8 B aligned

    if (threadIdx.x == 0) {
        for (int i = 0; i < Sw; ++i) {
            mbar_init(sm.wfull + 8 * i, 1);
            mbar_init(sm.wempty + 8 * i, 1);
        }
        for (int i = 0; i < Sx; ++i) {
            mbar_init(sm.xfull + 8 * i, 1);
            mbar_init(sm.xempty + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(sm.accfull + 8 * i, 1);
            mbar_init(sm.accempty + 8 * i, 128);
        }
        for (int w = 0; w < kSimtWarps; ++w) {  // attention ring barriers (the rings live in the X ring)
            for (int k = 0; k < kAttnSlots; ++k) mbar_init(smem_u32(attn_ctl + w * kAttnCtlBytes + 8 * k), 1);
            *reinterpret_cast<uint32_t*>(attn_ctl + w * kAttnCtlBytes + kAttnSlots * 8) = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        *w_progress = 0;
        *epi_count = 0;
        *n_live_s = p.batch;
    }
    const uint32_t acc_cols = (uint32_t)p.bpad;  // one accumulator, double-buffered
    uint32_t tmem_cols = 32;
    while (tmem_cols < 2 * acc_cols) tmem_cols *= 2;
    if (warp == 1) tmem_alloc(smem_u32(tmem_slot), tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------------ W producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            // L2 prefetch cursor, l2_ahead tiles ahead of the ring: HBM keeps
            // streaming future phases' weights into the 126 MB L2 while the ring
            // (a few tiles of shared memory) waits for barriers and activations.
            int ppi = -1, pk = 0, pe = 0;
            auto pf_next = [&]() {
                while (pk >= pe) {
                    if (++ppi >= p.n_phases) return;
                    if (prog[ppi].kind != kPhaseGemm) continue;
                    cta_range(prog[ppi], blk, G, pk, pe);
                }
                const Phase& q = prog[ppi];
                const int tile = pk / q.kb, k = pk - tile * q.kb;
                tma_prefetch_2d(p.maps + q.wmap, k * kBK, tile * kBM);
                ++pk;
            };
            for (int j = 0; j < p.l2_ahead; ++j) pf_next();
            uint32_t it = 0;
            for (int pi = 0; pi < p.n_phases; ++pi) {
                const Phase ph = prog[pi];
                if (ph.kind != kPhaseGemm) continue;
                const CUtensorMap* wm = p.maps + ph.wmap;
                int s, e;
                cta_range(ph, blk, G, s, e);
                for (int kbi = s; kbi < e; ++kbi, ++it) {
                    const uint32_t slot = it % Sw, ph_bit = (it / Sw) & 1u;
                    if (p.l2_ahead > 0 && ppi < p.n_phases) pf_next();
                    mbar_wait(sm.wempty + 8 * slot, ph_bit ^ 1u);
                    if (kbi == s) stamp(p, pi, 4);
                    if (kbi == e - 1) stamp(p, pi, 5);
                    const int tile = kbi / ph.kb, k = kbi - tile * ph.kb;
                    if (p.dbg & 4) {
                        mbar_arrive(sm.wfull + 8 * slot);
                    } else {
                        mbar_expect_tx(sm.wfull + 8 * slot, kWStageBytes);
                        tma_load_2d(sm.w + slot * kWStageBytes, wm, sm.wfull + 8 * slot, k * kBK, tile * kBM, pol);
                    }
                    *w_progress = it + 1;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer (whole warp, elected lane issues)
        const uint32_t idesc = idesc_bf16(kBM, p.bpad);
        uint32_t wit = 0, xit = 0, seg = 0;
        for (int pi = 0; pi < p.n_phases; ++pi) {
            const Phase ph = prog[pi];
            if (ph.kind != kPhaseGemm) continue;
            int s, e;
            cta_range(ph, blk, G, s, e);
            for (int kbi = s; kbi < e;) {
                const int tile = kbi / ph.kb;
                const int kend = min(e, (tile + 1) * ph.kb);
                const uint32_t a = seg & 1u, use = seg >> 1;
                mbar_wait(sm.accempty + 8 * a, (use & 1u) ^ 1u);
                tc_fence_after();
                const uint32_t d = tmem + a * acc_cols;
                for (int k = kbi; k < kend; ++k, ++wit, ++xit) {
                    const uint32_t ws = wit % Sw, xs = xit % Sx;
                    mbar_wait(sm.wfull + 8 * ws, (wit / Sw) & 1u);
                    mbar_wait(sm.xfull + 8 * xs, (xit / Sx) & 1u);
                    tc_fence_after();
                    const uint64_t da = smem_desc_sw128(sm.w + ws * kWStageBytes);
                    const uint64_t db = smem_desc_sw128(sm.x + xs * sm.xstage);
                    if (elect_one()) {
                        if (k == s) stamp(p, pi, 6);
                        if (k == e - 1) stamp(p, pi, 7);
                        const uint32_t acc0 = k > kbi ? 1u : 0u;
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk)
                            umma_bf16(d, da + (uint64_t)(2 * kk), db + (uint64_t)(2 * kk), idesc, kk ? 1u : acc0);
                        umma_commit(sm.wempty + 8 * ws);
                        umma_commit(sm.xempty + 8 * xs);
                    }
                    __syncwarp();
                }
                if (elect_one()) umma_commit(sm.accfull + 8 * a);
                __syncwarp();
                ++seg;
                kbi = kend;
            }
        }
    } else {
        // ------------------------------------------------------------------ warps 2..7
        const bool is_epi = warp >= 4;
        const int q = warp & 3;
        uint32_t xit = 0, seg = 0, gemm_done = 0;
        unsigned long long* ctr = reinterpret_cast<unsigned long long*>(p.bar + 2);
        const unsigned long long bar_base = p.bar_base;
        for (int pi = 0; pi < p.n_phases; ++pi) {
            const Phase ph = prog[pi];
            const bool gemm = ph.kind == kPhaseGemm;
            if (pi > 0) {
                const bool prev_gemm = prog[pi - 1].kind == kPhaseGemm;
                if (!prev_gemm) named_sync(1, kSimtThreads);  // this CTA's SIMT work of phase pi-1 is done
                else if (warp == 2 || is_epi) named_sync(2, 160);  // this CTA's epilogue of phase pi-1 is done
                if (warp == 2 && lane == 0) {
                    stamp(p, pi - 1, 3);
                    if (p.bar_mode == 0) counter_barrier(ctr, bar_base + (unsigned long long)pi * G);
                    else if (p.bar_mode == 1) grid_barrier(p.bar, p.bar + 1, (unsigned)G);
                    stamp(p, pi, 0);
                }
                __syncwarp();
                if (!gemm) named_sync(1, kSimtThreads);  // every CTA finished phase pi-1
            }
            const int n_live = *n_live_s;
            if (gemm) {
                int s, e;
                cta_range(ph, blk, G, s, e);
                if (warp == 2 && lane == 0) {
                    // X producer: this CTA's activation tiles, in MMA order
                    fence_proxy_async_global();
                    const uint64_t pol = policy_evict_last();
                    const CUtensorMap* xm = p.maps + ph.xmap;
                    for (int kbi = s; kbi < e; ++kbi, ++xit) {
                        const uint32_t slot = xit % Sx, ph_bit = (xit / Sx) & 1u;
                        mbar_wait(sm.xempty + 8 * slot, ph_bit ^ 1u);
                        const int k = kbi % ph.kb;
                        mbar_expect_tx(sm.xfull + 8 * slot, sm.xstage);
                        tma_load_2d(sm.x + slot * sm.xstage, xm, sm.xfull + 8 * slot, k * kBK, 0, pol);
                    }
                    stamp(p, pi, 1);
                } else if (is_epi) {
                    // epilogue: TMEM -> this CTA's partial slots (not gated by the barrier)
                    const int first_tile = s / ph.kb;
                    for (int kbi = s; kbi < e;) {
                        const int tile = kbi / ph.kb;
                        const int kend = min(e, (tile + 1) * ph.kb);
                        const uint32_t a = seg & 1u, use = seg >> 1;
                        mbar_wait(sm.accfull + 8 * a, use & 1u);
                        tc_fence_after();
                        const uint32_t taddr = tmem + a * acc_cols + ((uint32_t)(q * 32) << 16);
                        const int slot = tile - first_tile;
                        float* dst = p.partials + ((size_t)(blk * kMaxSeg + slot) * p.bpad) * kBM + q * 32 + lane;
                        for (int c0 = 0; c0 < p.bpad; c0 += 16) {
                            uint32_t r[16];
                            tmem_ld16_nowait(taddr + (uint32_t)c0, r);
                            tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 16; ++c) __stcg(dst + (size_t)(c0 + c) * kBM, __uint_as_float(r[c]));
                        }
                        tc_fence_before();
                        mbar_arrive(sm.accempty + 8 * a);
                        ++seg;
                        kbi = kend;
                    }
                    if (warp == 4 && lane == 0) stamp(p, pi, 2);
                }
                ++gemm_done;
            } else {
                switch (ph.kind) {
                    case kPhaseNorm: phase_norm(p, segtab, prog, ph, live, n_live, red); break;
                    case kPhaseAttn:
                        phase_attn(p, segtab, prog[ph.src], ph.layer, live, n_live, scratch, attn_ctl);
                        break;
                    case kPhaseAct: phase_act(p, segtab, prog[ph.src], n_live); break;
                    case kPhaseHeadReduce: phase_head_reduce(p, segtab, prog[ph.src], n_live); break;
                    case kPhaseDecide: {
                        float4* merged = reinterpret_cast<float4*>(scratch);  // X ring is idle
                        decide_merge(p, (prog[ph.src].tiles + kHeadChunk - 1) / kHeadChunk, n_live, merged);
                        named_sync(3, kSimtThreads);
                        if (warp == 2) phase_decide(p, ph, merged, live, n_live_s);
                        break;
                    }
                    case kPhaseFinalize: phase_finalize(p, red); break;
                    default: break;
                }
            }
        }
        if (prog[p.n_phases - 1].kind != kPhaseGemm) named_sync(1, kSimtThreads);
        else if (warp == 2 || is_epi) named_sync(2, 160);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, tmem_cols);
    }
}

}  // namespace

void launch(const Params& p, const int4* segtab, int grid, cudaStream_t s) {
    const unsigned smem = smem_bytes(p.bpad, p.w_stages, p.x_stages, p.n_phases, p.n_segtab);
    EEB_CUDA(cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    EEB_CUDA(cudaLaunchKernelEx(&cfg, step_kernel, p, segtab));
}

}  // namespace mk
}  // namespace eeb
