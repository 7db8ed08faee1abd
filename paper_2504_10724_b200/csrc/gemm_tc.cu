// gemm_tc.cu — tier-2 decode GEMM on the 5th-generation tensor cores.
//
// y[B, N] = x[B, K] · W[N, K]^T for bf16 weights once the batch makes the
// weight stream a dense contraction (B >= 16: 2·B flop per weight byte
// outruns the CUDA cores, SURVEY §7 hard part 6).  Swap-AB: the weight tile is
// the MMA's M operand (128 output features), the batch is its N operand, so a
// [128 x B] f32 accumulator lives in TMEM and one tcgen05.mma
// (M=128, N=B, K=16) consumes a 128 x 16 weight slice.
//
// Warp roles (192 threads, one CTA per SM):
//   warp 0      TMA producer: weight tile [128 x 64] + activation tile [B x 64]
//               per stage, 128B-swizzled, arriving on the stage's mbarrier;
//   warp 1      TMEM allocator + single-thread MMA issuer; tcgen05.commit
//               frees a stage and, after the last k-block, signals the epilogue;
//   warps 2..5  epilogue: tcgen05.ld 32x32b (thread = output feature), fused
//               residual-add / ReLU / SwiGLU / f32 store, or split-K partials.
// Split-K spreads small N over the 148 SMs; partials are reduced in a fixed
// order by splitk_epilogue (deterministic, no atomics).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cooperative_groups.h>

#include <cstdlib>
#include <mutex>

#include "kernels.h"

namespace eeb {

namespace {

constexpr int kBM = 128;           // output features per tile (UMMA M)
constexpr int kRS = kBM + 4;         // row stride (floats) of a staged cs > 1 partial: 16-B aligned rows
constexpr int kBK = 64;            // K per stage: one 128-byte swizzle atom of bf16
constexpr int kThreads = 192;
constexpr int kSmemBudget = 227 * 1024;

// ---- PTX wrappers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
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
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128B-swizzled shared-memory matrix descriptor (rows of 128 B,
// 8-row atoms 1024 B apart).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);  // start address
    d |= (uint64_t)1 << 16;                    // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;          // stride byte offset: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
    return d;
}
// Instruction descriptor: kind::f16, A = B = bf16, D = f32, both K-major.
__host__ __device__ constexpr uint32_t instr_desc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Two 16-column TMEM loads in flight before one wait (epilogue latency).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr + 16u));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ bool elect_one_sync() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

namespace cg = cooperative_groups;

struct TcParams {
    int cs;            // CTAs per cluster along the split dimension (1 = no on-chip reduction)
    int N, K;
    int kb_per;        // k-blocks per split
    int kblocks;       // total k-blocks
    int bpad;          // UMMA N (batch rows per CTA, multiple of 16)
    int rh;            // row blocks: CTA x = m_tile * rh + block; block b covers rows [b bpad, (b + 1) bpad)
    int stages;
    int tmem_cols;
    const int* n_active;
    float* part;       // split-K planes, row stride N
    int64_t split_stride;
    __nv_bfloat16* act_out;  // fused MLP activation (splits == 1): bf16 [rows][N or N/2]
    int act_kind;            // 1 ReLU, 2 SwiGLU over interleaved (gate, up) features
    float4* head_tri;  // exit-head epilogue (splits == 1): per (row, tile) {max, sumexp, argmax}
    int tiles;
    int vocab_off;     // added to the argmax (vocab-parallel shard)
    const char* pf;    // next GEMM's weights: L2 prefetch, this CTA's share
    size_t pf_bytes;
    unsigned long long* trace;  // timing experiments: 8 globaltimer stamps per CTA (null = off)
    int dbg;                    // timing experiments: bit 0 = no plane stores (results wrong)
    int skip_dead;              // read n_active before the weight prefetch (skip it when 0)
    int l2pf;                   // L2-prefetch the weight tiles beyond the smem stages before the PDL wait
    int tma_out;                // split-K planes written by a TMA store of the smem-staged tile (tmap_o)
    int orows, obufs;           // rows per TMA store chunk, smem buffers (1 or 2)
    Stamp st;                   // in-graph launch timeline (eeb_debug_stamps)
};

// Timeline stamps are compiled in only for the timing experiments
// (-DEEB_GEMM_TRACE, tools/gemm_trace.py); the product kernel has none.
#ifdef EEB_GEMM_TRACE
#define EEB_STAMP(cond, slot) \
    do {                      \
        if (tr && (cond)) tr[slot] = gtime(); \
    } while (0)
#else
#define EEB_STAMP(cond, slot) \
    do {                      \
    } while (0)
#endif
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
    return t;
}

// kCsF: the instantiations for 2- and 4-CTA clusters (the on-chip K
// reduction of the fused up projection with 16-byte DSMEM loads); their
// extra registers stay out of the plane GEMMs' instantiation (kCsF = 0:
// no cluster, or any other cluster size through the scalar path).
template <int kCsF>
__global__ void __launch_bounds__(kThreads, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
                   const __grid_constant__ CUtensorMap tmap_o, TcParams p) {
    StampScope stamp_scope(p.st);
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzle atoms.
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* base_ptr = smem_raw + (base - raw);
    const int S = p.stages;
    const uint32_t a_bytes = kBM * kBK * 2;
    const uint32_t b_bytes = (uint32_t)p.bpad * kBK * 2;
    const uint32_t stage_bytes = a_bytes + b_bytes;
    // barriers + tmem slot after the tiles
    uint64_t* bars = reinterpret_cast<uint64_t*>(base_ptr + (size_t)S * stage_bytes);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S), tfull = smem_u32(bars + 2 * S);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m_tile = blockIdx.x / p.rh, split = blockIdx.y;
    const int r_off = (blockIdx.x % p.rh) * p.bpad;  // this CTA's first batch row
    const int kb0 = split * p.kb_per;
    const int kb1 = min(kb0 + p.kb_per, p.kblocks);
    const int nkb = kb1 - kb0;

#ifdef EEB_GEMM_TRACE
    unsigned long long* tr = p.trace ? p.trace + 8 * ((size_t)blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
#endif
    EEB_STAMP(threadIdx.x == 0, 0);  // CTA start
    pdl_launch_dependents();  // let the next kernel of the step get resident and prefetch
    __shared__ int pre_s;
    if (threadIdx.x == 0) {
        // The live-row hint is loaded first (its latency overlaps the barrier
        // inits).  No weight prefetch when no row is live (all exited): read
        // before the PDL wait it may be stale, which costs only a useless or a
        // missed prefetch — the count after the wait decides what is computed.
        const int hint = p.skip_dead ? *reinterpret_cast<const volatile int*>(p.n_active) - r_off : 1;
        prefetch_tmap(&tmap_w);
        prefetch_tmap(&tmap_x);
        if (p.tma_out) prefetch_tmap(&tmap_o);
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(tfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // Weights do not depend on the previous kernel: the first stages' weight
        // tiles stream before the TMEM allocation and the PDL wait; the
        // activation tiles follow once the predecessor's output is visible.
        const int pre = hint <= 0 ? 0 : min(S, nkb);
        const uint64_t pol_w0 = policy_evict_first();
        for (int i = 0; i < pre; ++i) {
            const uint32_t sa = base + (uint32_t)i * stage_bytes;
            mbar_expect_tx(full0 + 8 * i, stage_bytes);
            tma_load_2d(sa, &tmap_w, full0 + 8 * i, (kb0 + i) * kBK, m_tile * kBM, pol_w0);
        }
        // the rest of this CTA's weight tiles -> L2, also before the wait: a
        // CTA resident while a latency-bound predecessor (norm) runs streams
        // its whole share then, and its later stages load from L2
        if (p.l2pf && hint > 0)
            for (int i = pre; i < nkb; ++i)
                asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                                 reinterpret_cast<uint64_t>(&tmap_w)),
                             "r"((kb0 + i) * kBK), "r"(m_tile * kBM)
                             : "memory");
        pre_s = pre;
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"((uint32_t)p.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    EEB_STAMP(threadIdx.x == 0, 1);  // barriers + TMEM ready

    if (warp == 0) {
        const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
        const int pre = pre_s;  // weight stages already in flight (issued by thread 0 above)
#ifdef EEB_L2_PREFETCH
        // (compiled in only for the experiment: measured slower, see gemm_tc host)
        if (lane != 0 && p.pf_bytes) {
            // lanes 1..31, behind this CTA's own first tiles: its share of the
            // next GEMM's weights -> L2
            const size_t nct = (size_t)gridDim.x * gridDim.y;
            const size_t cta = (size_t)blockIdx.y * gridDim.x + blockIdx.x;
            const size_t share = ((p.pf_bytes + nct - 1) / nct + 15) & ~(size_t)15;
            const size_t b0 = cta * share, b1 = min(p.pf_bytes, b0 + share);
            constexpr size_t kPiece = 16384;
            for (size_t o = b0 + (size_t)(lane - 1) * kPiece; o < b1; o += 31 * kPiece) {
                const uint32_t n = (uint32_t)min(kPiece, b1 - o) & ~15u;
                if (n)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.pf + o), "r"(n) : "memory");
            }
        }
#endif
        if (lane == 0) {
            pdl_wait();
            stamp_waited(p.st);
            EEB_STAMP(true, 2);  // predecessor complete
            for (int i = 0; i < pre; ++i)
                tma_load_2d(base + (uint32_t)i * stage_bytes + a_bytes, &tmap_x, full0 + 8 * i, (kb0 + i) * kBK, r_off,
                            pol_x);
            // every row exited before this layer: complete the stages already
            // in flight (their barriers expect the X bytes too) and stream no
            // more (read after the X loads are issued: off the critical path)
            const int last = *p.n_active - r_off > 0 ? nkb : pre;
            if (last == pre)
                for (int i = 0; i < pre; ++i) mbar_wait(full0 + 8 * i, 0);
            for (int i = pre; i < last; ++i) {
                const int s = i % S;
                const uint32_t ph = (uint32_t)(i / S) & 1u;
                mbar_wait(empty0 + 8 * s, ph ^ 1u);
                const uint32_t sa = base + (uint32_t)s * stage_bytes;
                mbar_expect_tx(full0 + 8 * s, stage_bytes);
                const int kc = (kb0 + i) * kBK;
                tma_load_2d(sa, &tmap_w, full0 + 8 * s, kc, m_tile * kBM, pol_w);
                tma_load_2d(sa + a_bytes, &tmap_x, full0 + 8 * s, kc, r_off, pol_x);
            }
        }
        __syncwarp();  // reconverge before the CTA barrier (bar.sync is warp-aligned)
    } else if (warp == 1) {
        // The whole warp runs the loop (descriptors stay warp-uniform: uniform
        // registers, no per-op R2UR) and one elected lane issues — a
        // single-lane loop issues tcgen05.mma several times slower.
        const uint32_t idesc = instr_desc(kBM, p.bpad);
        pdl_wait();
        const int live = *p.n_active - r_off;  // <= 0: every row of this block exited, nothing to multiply
        for (int i = 0; i < (live > 0 ? nkb : 0); ++i) {
            const int s = i % S;
            const uint32_t ph = (uint32_t)(i / S) & 1u;
            mbar_wait(full0 + 8 * s, ph);
            tc_fence_after();
            EEB_STAMP(i == 0 && lane == 0, 3);  // first stage (W + X) landed
            const uint32_t sa = base + (uint32_t)s * stage_bytes;
            const uint64_t da = smem_desc(sa), db = smem_desc(sa + a_bytes);
            if (elect_one_sync()) {
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k)  // +32 B per K=16 step inside the swizzle atom
                    umma(tmem, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k), idesc, (i | k) != 0);
                umma_commit(empty0 + 8 * s);
            }
            __syncwarp();
        }
        if (live > 0 && elect_one_sync()) umma_commit(tfull);
        __syncwarp();
    } else {
        // epilogue: warp w reads TMEM lanes 32*(w%4) .. +31  (thread = output feature)
        const int quarter = warp & 3;
        const int n = m_tile * kBM + quarter * 32 + lane;
        pdl_wait();  // n_active and the plane workspace belong to the previous kernels
        const int rows = *p.n_active - r_off;  // this CTA's live rows (<= 0: none)
        if (rows > 0) {
        mbar_wait(tfull, 0);
        tc_fence_after();
        if (threadIdx.x == 64) stamp_mark(p.st);  // accumulator complete (timeline)
        EEB_STAMP(threadIdx.x == 64, 4);  // accumulator complete
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16);
        if (p.head_tri && p.cs == 1) {
            // Fused exit-head tail: stage the [rows x 128 vocab] logits tile
            // transposed in the drained pipeline smem, then two threads per row
            // scan 64 entries each for max / first argmax / sum exp(l - max).
            float* red = reinterpret_cast<float*>(base_ptr);
            const int f = quarter * 32 + lane;
            for (int c0 = 0; c0 < min(rows, p.bpad); c0 += 16) {  // live rows only
                float v[16];
                tmem_ld16(taddr + (uint32_t)c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) red[(c0 + j) * (kBM + 1) + f] = v[j];
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int t = threadIdx.x - 64, hf = t & 1;
            const int n0 = m_tile * kBM + hf * 64;
            const int nv = max(0, min(64, p.N - n0));
            const int lim = min(rows, p.bpad);
            for (int r0 = 0; r0 < lim; r0 += 64) {  // warp-uniform trip count (shuffles below)
                const int r = r0 + (t >> 1);
                const int nvr = r < lim ? nv : 0;
                const float* src = red + min(r, p.bpad - 1) * (kBM + 1) + hf * 64;
                float m = -INFINITY;
                int am = 0x7fffffff;
                for (int j = 0; j < nvr; ++j)
                    if (src[j] > m) { m = src[j]; am = n0 + j; }
                float sum = 0.f;
                for (int j = 0; j < nvr; ++j) sum += __expf(src[j] - m);
                const float m2 = __shfl_xor_sync(0xffffffffu, m, 1);
                const int a2 = __shfl_xor_sync(0xffffffffu, am, 1);
                const float s2 = __shfl_xor_sync(0xffffffffu, sum, 1);
                const float M = fmaxf(m, m2);
                const int A = (m2 > m || (m2 == m && a2 < am)) ? a2 : am;
                const float S = (m == -INFINITY ? 0.f : sum * __expf(m - M)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - M));
                if (hf == 0 && r < lim)
                    p.head_tri[(int64_t)(r + r_off) * p.tiles + m_tile] = make_float4(M, S, __int_as_float(A + p.vocab_off), 0.f);
            }
        } else if (p.act_out && p.cs == 1) {
            // Fused MLP activation: the up projection's tile goes straight to the
            // down GEMM's bf16 input — no split-K planes, no activation kernel.
            const int lim = min(rows, p.bpad);
            for (int c0 = 0; c0 < min(rows, p.bpad); c0 += 16) {  // live rows only
                float v[16];
                tmem_ld16(taddr + (uint32_t)c0, v);  // warp-collective
                if (p.act_kind == 2) {
                    const int half_n = p.N / 2;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const float u = __shfl_xor_sync(0xffffffffu, v[j], 1);  // odd lane: up, even: gate
                        if ((lane & 1) == 0 && n < p.N && c0 + j < lim) {
                            const float g = v[j];
                            p.act_out[(int64_t)(c0 + j + r_off) * half_n + n / 2] = __float2bfloat16_rn(g / (1.f + __expf(-g)) * u);
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (n < p.N && c0 + j < lim)
                            p.act_out[(int64_t)(c0 + j + r_off) * p.N + n] = __float2bfloat16_rn(fmaxf(v[j], 0.f));
                }
            }
        } else if (p.cs == 1 && p.tma_out) {
            // Split-K plane through shared memory: the [rows][128] f32 tile is
            // staged in the drained pipeline stages (thread = feature: each row
            // is 32 consecutive floats per warp, conflict-free) and written by
            // one TMA bulk tensor store — per-thread global stores of the
            // same 32 KB cost ~2.4 us of the GEMM's tail (measured in the C2 step).
            // Large row counts (prefill chunks, batch >= 128) go in chunks of
            // p.orows rows through two alternating smem buffers.
            const int f = quarter * 32 + lane;
            const int lim = min(rows, p.bpad);
            const int OR = p.orows;
            const uint32_t buf_floats = (uint32_t)OR * kBM;
            for (int r0 = 0, b = 0; r0 < lim; r0 += OR, b ^= 1) {
                float* stg = reinterpret_cast<float*>(base_ptr) + (p.obufs > 1 ? b * buf_floats : 0);
                if (r0 > 0 && (r0 >= 2 * OR || p.obufs == 1)) {  // this buffer's previous store has read its smem
                    if (threadIdx.x == 64) {
                        if (p.obufs > 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                }
                const int rend = min(lim, r0 + OR);
                int c0 = r0;
                for (; c0 + 32 <= r0 + OR && c0 < rend; c0 += 32) {
                    float v[32];
                    tmem_ld32(taddr + (uint32_t)c0, v);  // warp-collective
#pragma unroll
                    for (int j = 0; j < 32; ++j) stg[(c0 - r0 + j) * kBM + f] = v[j];
                }
                for (; c0 < rend; c0 += 16) {
                    float v[16];
                    tmem_ld16(taddr + (uint32_t)c0, v);
#pragma unroll
                    for (int j = 0; j < 16; ++j) stg[(c0 - r0 + j) * kBM + f] = v[j];
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> TMA reads
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (threadIdx.x == 64) {
                    asm volatile(
                        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                            reinterpret_cast<uint64_t>(&tmap_o)),
                        "r"(m_tile * kBM), "r"(r0 + r_off), "r"(split), "r"(smem_u32(stg))
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
            if (threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // written before the grid completes
        } else if (p.cs == 1) {
            float* plane = p.part + (int64_t)split * p.split_stride;
            // only the live rows' columns (warp-uniform bound), 32 per wait
            const int lim = min(rows, p.bpad);
            int c0 = 0;
            for (; c0 + 32 <= p.bpad && c0 < lim; c0 += 32) {
                float v[32];
                tmem_ld32(taddr + (uint32_t)c0, v);  // warp-collective
                if (n < p.N && !(p.dbg & 1)) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (c0 + j < lim) plane[(int64_t)(c0 + j + r_off) * p.N + n] = v[j];
                }
            }
            for (; c0 < lim; c0 += 16) {
                float v[16];
                tmem_ld16(taddr + (uint32_t)c0, v);
                if (n < p.N && !(p.dbg & 1)) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (c0 + j < lim) plane[(int64_t)(c0 + j + r_off) * p.N + n] = v[j];
                }
            }
        } else {
            // stage this CTA's [128 features][bpad rows] partial in its (now idle) pipeline smem
            float* red = reinterpret_cast<float*>(base_ptr);
            const int f = quarter * 32 + lane;
            for (int c0 = 0; c0 < min(rows, p.bpad); c0 += 16) {  // live rows only
                float v[16];
                tmem_ld16(taddr + (uint32_t)c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) red[(c0 + j) * kRS + f] = v[j];
            }
        }
        }  // rows > 0
    }
    // every thread: the live-row count (uniform over a cluster) gates the on-chip reduction
    pdl_wait();
    const int rows_all = *p.n_active - r_off;  // (r_off is uniform over a cluster: clusters run along K)
    if (p.cs > 1 && rows_all > 0) {
        // Split-K reduction on chip: the cs CTAs of a cluster hold consecutive
        // k-ranges of one tile; CTA rank r sums rows r, r+cs, ... of the tile
        // over the cluster's smem partials in rank (= k) order (deterministic)
        // and finishes them: one plane per cluster (cs x fewer partial planes
        // for the consumers to read), or the fused MLP activation, or the
        // exit-head softmax partials — the fused epilogues get the SM coverage
        // of split-K without a round trip through HBM/L2.
        cg::cluster_group cluster = cg::this_cluster();
        // partials staged (st.shared) -> visible to the cluster: release/acquire
        // barrier (no cg::sync, whose GPU-scope fence would also drain this
        // CTA's global stores)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        EEB_STAMP(threadIdx.x == 64, 7);  // cluster partials visible
        const int rank = (int)cluster.block_rank();
        const int lim = min(rows_all, p.bpad);  // (not re-read: an L2 round trip after the barrier's L1 flush)
        const float* red = reinterpret_cast<const float*>(base_ptr);
        // this rank's finished rows (head mode), after the staged partials
        float* fin = reinterpret_cast<float*>(base_ptr) + (size_t)p.bpad * kRS;
        if (warp >= 2) {
            const int t = threadIdx.x - 64;  // 0..127: feature of the tile
            const int n = m_tile * kBM + t;
            float* plane = p.part + (int64_t)(split / p.cs) * p.split_stride;
            const float* peer[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) peer[q] = cluster.map_shared_rank(red, q < p.cs ? q : 0);
            auto finish = [&](int j, int row, float acc) {
                if (p.head_tri) {
                    fin[j * kRS + t] = acc;
                } else if (p.act_out) {
                    if (p.act_kind == 2) {
                        const float u = __shfl_xor_sync(0xffffffffu, acc, 1);  // odd lane: up, even: gate
                        if ((t & 1) == 0 && n < p.N)
                            p.act_out[(int64_t)(row + r_off) * (p.N / 2) + n / 2] = __float2bfloat16_rn(acc / (1.f + __expf(-acc)) * u);
                    } else if (n < p.N) {
                        p.act_out[(int64_t)(row + r_off) * p.N + n] = __float2bfloat16_rn(fmaxf(acc, 0.f));
                    }
                } else if (n < p.N) {
                    plane[(int64_t)(row + r_off) * p.N + n] = acc;
                }
            };
            // kR rows x cs peers of DSMEM loads in flight at once (a
            // row-at-a-time loop pays one DSMEM round trip per load);
            // warp-uniform trip counts (the SwiGLU pairing shuffles).  The
            // 4-CTA clusters of the decode up projection: 16 rows x 4 peers,
            // a 64-row tile in one DSMEM round trip per rank.
            if (kCsF == 2 || kCsF == 4) {
                // 16-byte DSMEM loads (DSMEM moves ~20 B/clk per SM; per-thread
                // 4-byte loads took 2.7 us for the 64-row tile): lane = 4
                // consecutive features, epilogue warp ew takes this rank's
                // rows j = ew, ew + 4, ...; kJ rows x kCsF peers in flight.
                constexpr int C = kCsF == 4 ? 4 : 2;
                const int ew = warp - 2, n4 = m_tile * kBM + 4 * lane;
                constexpr int kJ = 4;
                for (int j0 = ew; rank + j0 * C < lim; j0 += 4 * kJ) {
                    float4 v[kJ][C];
#pragma unroll
                    for (int r = 0; r < kJ; ++r) {
                        const int row = rank + (j0 + 4 * r) * C;
#pragma unroll
                        for (int q = 0; q < C; ++q)
                            v[r][q] = row < lim ? *reinterpret_cast<const float4*>(peer[q] + row * kRS + 4 * lane)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int r = 0; r < kJ; ++r) {
                        const int j = j0 + 4 * r, row = rank + j * C;
                        if (row >= lim) break;
                        float4 a = v[r][0];  // rank (= k) order, as the scalar path
#pragma unroll
                        for (int q = 1; q < C; ++q) {
                            a.x += v[r][q].x;
                            a.y += v[r][q].y;
                            a.z += v[r][q].z;
                            a.w += v[r][q].w;
                        }
                        if (p.head_tri) {
                            *reinterpret_cast<float4*>(fin + j * kRS + 4 * lane) = a;
                        } else if (n4 < p.N) {
                            if (p.act_out && p.act_kind == 2) {  // (gate, up) pairs -> 2 outputs
                                const __nv_bfloat162 o = __floats2bfloat162_rn(a.x / (1.f + __expf(-a.x)) * a.y,
                                                                               a.z / (1.f + __expf(-a.z)) * a.w);
                                *reinterpret_cast<__nv_bfloat162*>(p.act_out + (int64_t)(row + r_off) * (p.N / 2) + n4 / 2) = o;
                            } else if (p.act_out) {
                                const __nv_bfloat162 lo = __floats2bfloat162_rn(fmaxf(a.x, 0.f), fmaxf(a.y, 0.f));
                                const __nv_bfloat162 hi = __floats2bfloat162_rn(fmaxf(a.z, 0.f), fmaxf(a.w, 0.f));
                                uint2 u;
                                u.x = *reinterpret_cast<const uint32_t*>(&lo);
                                u.y = *reinterpret_cast<const uint32_t*>(&hi);
                                *reinterpret_cast<uint2*>(p.act_out + (int64_t)(row + r_off) * p.N + n4) = u;
                            } else {
                                *reinterpret_cast<float4*>(plane + (int64_t)(row + r_off) * p.N + n4) = a;
                            }
                        }
                    }
                }
            } else {
                constexpr int kR = 4;
                for (int j0 = 0; rank + j0 * p.cs < lim; j0 += kR) {
                    float v[kR][8];
#pragma unroll
                    for (int r = 0; r < kR; ++r) {
                        const int row = rank + (j0 + r) * p.cs;
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            v[r][q] = (q < p.cs && row < lim) ? peer[q][row * kRS + t] : 0.f;
                    }
#pragma unroll
                    for (int r = 0; r < kR; ++r) {
                        const int j = j0 + r;
                        const int row = rank + j * p.cs;
                        if (row >= lim) break;
                        float acc = 0.f;
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (q < p.cs) acc += v[r][q];
                        finish(j, row, acc);
                    }
                }
            }
        }
        // keep every CTA's partial alive until the whole cluster has read it: the
        // DSMEM loads have returned (their values were used), so a relaxed
        // arrive suffices and the act/plane stores above need not drain
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
        if (p.head_tri && warp >= 2) {
            // two threads per finished row scan 64 vocab entries each
            const int t = threadIdx.x - 64, hf = t & 1;
            const int n0 = m_tile * kBM + hf * 64;
            const int nv = max(0, min(64, p.N - n0));
            const int nmine = lim > rank ? (lim - rank + p.cs - 1) / p.cs : 0;
            for (int j0 = 0; j0 < nmine; j0 += 64) {
                const int j = j0 + (t >> 1);
                const int nvr = j < nmine ? nv : 0;
                const float* src = fin + min(j, max(nmine - 1, 0)) * kRS + hf * 64;
                float m = -INFINITY;
                int am = 0x7fffffff;
                for (int q = 0; q < nvr; ++q)
                    if (src[q] > m) { m = src[q]; am = n0 + q; }
                float sum = 0.f;
                for (int q = 0; q < nvr; ++q) sum += __expf(src[q] - m);
                const float m2 = __shfl_xor_sync(0xffffffffu, m, 1);
                const int a2 = __shfl_xor_sync(0xffffffffu, am, 1);
                const float s2 = __shfl_xor_sync(0xffffffffu, sum, 1);
                const float M = fmaxf(m, m2);
                const int A = (m2 > m || (m2 == m && a2 < am)) ? a2 : am;
                const float S = (m == -INFINITY ? 0.f : sum * __expf(m - M)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - M));
                const int row = rank + j * p.cs;
                if (hf == 0 && j < nmine)
                    p.head_tri[(int64_t)(row + r_off) * p.tiles + m_tile] = make_float4(M, S, __int_as_float(A + p.vocab_off), 0.f);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    EEB_STAMP(threadIdx.x == 0, 5);  // epilogue stores issued
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)p.tmem_cols));
        EEB_STAMP(lane == 0, 6);  // TMEM released
    }
}

// ---- host side -----------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

CUtensorMap make_map(const void* ptr, int rows, int cols, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(5, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

}  // namespace

bool gemm_tc_available() { return encode_fn() != nullptr; }

// Smallest batch the tensor-core tier takes.  Rows are padded to UMMA N = 16
// (the padding costs MMA issue slots only; the weight stream is the same) and
// the tcgen05 path prefetches its weights before the PDL wait, which the
// CUDA-core GEMV does not: measured at batch 1 (C2, tools/b1check.py) a full
// 24-layer step takes 1.09 ms on tcgen05 vs 1.39 ms on the GEMV, an exit-6
// step 0.45 vs 0.48 ms.  EEB_TC_MIN_ROWS overrides (A/B against the GEMV).
int tc_min_rows() {
    static const int v = std::getenv("EEB_TC_MIN_ROWS") ? std::max(1, std::atoi(std::getenv("EEB_TC_MIN_ROWS"))) : 1;
    return v;
}

void make_bf16_map(void* out_map, const void* ptr, int rows, int cols, int box_rows) {
    if (!encode_fn()) throw Error(5, "cuTensorMapEncodeTiled unavailable");
    *static_cast<CUtensorMap*>(out_map) = make_map(ptr, rows, cols, box_rows);
}

void make_kv_tensor_map(void* out_map, const void* base, int head_dim, int max_seq, int slots_x_heads,
                        int box_rows) {
    if (!encode_fn()) throw Error(5, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[3] = {(cuuint64_t)head_dim, (cuuint64_t)max_seq, (cuuint64_t)slots_x_heads};
    const cuuint64_t strides[2] = {(cuuint64_t)head_dim * 2, (cuuint64_t)head_dim * 2 * max_seq};
    const cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(static_cast<CUtensorMap*>(out_map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(5, "cuTensorMapEncodeTiled (kv) failed: " + std::to_string((int)r));
}

int gemm_tc(const GemmArgs& a, cudaStream_t s) {
    if (a.dtype != 1 || a.max_rows < tc_min_rows() || a.max_rows > 256 || a.K % kBK != 0) return 0;
    if (!gemm_tc_available()) return 0;
    int bpad = (a.max_rows + 15) / 16 * 16;
    const int tiles = (a.N + kBM - 1) / kBM;
    // more than 128 rows (large decode batches) on plain split-K GEMMs: two
    // CTAs per weight tile, 128 rows each (adjacent CTAs: the second read of
    // the tile hits L2), so each CTA keeps 3 pipeline stages and a 128-column
    // accumulator and the split count halves (longer K per CTA)
    static const bool env_rhalf = !std::getenv("EEB_TC_RHALF") || std::atoi(std::getenv("EEB_TC_RHALF")) != 0;
    // ... except for long K (>= 128 k-blocks: the 34B / 70B layer shapes): one
    // CTA per weight tile over all rows (one 256-column accumulator, the tile
    // read once), 4 stages, one CTA per SM, splits filling one wave of SMs —
    // measured (tools/gemm_split_sweep.py, B=256, 34B QKV / O / up / down):
    // 60.7 / 36.7 / 195 / 93.4 us -> 46.4 / 33.4 / 177.6 / 82.7 us; C2's
    // K = 2048 shapes keep the row halves (equal or better there)
    static const bool env_deep = !std::getenv("EEB_TC_DEEP") || std::atoi(std::getenv("EEB_TC_DEEP")) != 0;
    const bool deep = env_deep && bpad > 128 && a.K / kBK >= 128 && !a.head_tri && !a.act_out;
    const int rh = env_rhalf && bpad > 128 && !deep ? (bpad + 127) / 128 : 1;
    if (rh > 1) bpad = 128;
    const int mt = tiles * rh;  // CTAs per split
    const int kblocks = a.K / kBK;
    // split K so the grid covers the SMs once, keeping >= 2 k-blocks per CTA
    static const int env_wave = std::getenv("EEB_TC_WAVE") ? std::atoi(std::getenv("EEB_TC_WAVE")) : 0;
    static const int env_stages = std::getenv("EEB_TC_STAGES") ? std::atoi(std::getenv("EEB_TC_STAGES")) : 0;
    const int wave = env_wave > 0 ? env_wave : (deep ? 1 : 2) * a.num_sms;  // co-resident CTAs per SM
    // (at most 16 planes: the attention kernels sum up to 16 QKV planes in registers;
    //  only narrow GEMMs such as a 70B tensor-parallel QKV shard would want more)
    int splits = std::max(1, std::min(std::min(kblocks / 2, wave / mt), 16));
    static const int env_widesplit = std::getenv("EEB_TC_WIDESPLIT") ? std::atoi(std::getenv("EEB_TC_WIDESPLIT")) : 2;
    if (mt > wave / 2 && !a.head_tri && !a.act_out) {
        // wide GEMMs (more tiles than half a wave, e.g. the 34B up projection:
        // 344 tiles): the split count with the best wave efficiency, planes
        // capped at the weight bytes (s * rows * 4 <= K * 2)
        // (deep tiles: up to 3 splits, each extra split must gain 0.1 of wave
        //  efficiency — 34B QKV 80 tiles: 3 splits; up 344 tiles: 2)
        double best = 0.0;
        const int max_sp = deep ? std::max(env_widesplit, 3) : env_widesplit;
        const double gain = deep ? 0.1 : 0.02;
        for (int sp = 1; sp <= max_sp && sp <= kblocks / 2 && (size_t)sp * bpad * 4 <= (size_t)a.K * 2; ++sp) {
            const int units = mt * sp;
            const double eff = (double)units / ((double)((units + wave - 1) / wave) * wave);
            if (eff > best + gain) {
                best = eff;
                splits = sp;
            }
        }
    }
    // many rows (prefill chunks): cap the f32 partial planes at about the
    // weight bytes (splits * rows * N * 4 <= N * K * 2); decode shapes are
    // unaffected (C2: K / (2 * 64) = 16 >= the splits chosen above)
    // (opt-in EEB_TC_PLANECAP=1: measured 126 vs 125 ms for the C2 prefill)
    static const bool plane_cap = std::getenv("EEB_TC_PLANECAP") && std::atoi(std::getenv("EEB_TC_PLANECAP")) != 0;
    if (plane_cap) splits = std::max(1, std::min(splits, a.K / (2 * bpad)));
    // at most 12 planes: fewer partial planes for the consumer (residual norm,
    // attention) to sum against a slightly longer K per CTA — measured
    // ms/step 16 -> 12: C2 B=64 1.341 -> 1.314, B=16 1.183 -> 1.166, B=256
    // 2.262 -> 2.257, 34B flat-12 B=64 3.220 -> 3.161 (10: no better)
    static const int env_maxsplit = std::getenv("EEB_TC_MAXSPLIT") ? std::atoi(std::getenv("EEB_TC_MAXSPLIT")) : 12;
    if (env_maxsplit > 0) splits = std::min(splits, env_maxsplit);
    // (sweeps only: EEB_TC_SPLITS forces the split count of plain split-K GEMMs)
    static const int env_splits = std::getenv("EEB_TC_SPLITS") ? std::atoi(std::getenv("EEB_TC_SPLITS")) : 0;
    if (env_splits > 0 && !a.head_tri && !a.act_out) splits = std::max(1, std::min(env_splits, kblocks / 2));
    int kb_per = (kblocks + splits - 1) / splits;
    splits = (kblocks + kb_per - 1) / kb_per;
    // Clusters of cs CTAs along K reduce their partials on chip (DSMEM): pick
    // the largest cs <= 8 dividing the split count.
    static const int env_cs = std::getenv("EEB_TC_CLUSTER") ? std::atoi(std::getenv("EEB_TC_CLUSTER")) : 1;
    int cs = 1;
    for (int c = std::min(env_cs, 8); c > 1; --c)
        if (splits % c == 0) {
            cs = c;
            break;
        }
    if (a.head_tri || a.act_out) {
        // The fused epilogues need whole-K tiles: one CTA per tile, or a
        // cluster of cs CTAs splitting K whose partials are reduced on chip
        // (DSMEM) so that the grid still covers the SMs.
        // measured (C2): the up projection gains from clustering (64 tiles ->
        // 4-CTA clusters), the exit head does not; EEB_ACT_CS / EEB_HEAD_CS override.
        static const int env_act_cs = std::getenv("EEB_ACT_CS") ? std::atoi(std::getenv("EEB_ACT_CS")) : -1;
        static const int env_head_cs = std::getenv("EEB_HEAD_CS") ? std::atoi(std::getenv("EEB_HEAD_CS")) : 1;
        const int env_fcs = a.head_tri ? env_head_cs : env_act_cs;
        // cs: the best wave efficiency tiles*cs / (waves * wave), near-ties to
        // the smaller cluster (fewer CTAs, longer K each).  Activations: cs in
        // {1, 2, 4} (the 2- and 4-CTA clusters have the vectorised DSMEM
        // reduction; with the scalar one, B=64: 80 tiles x K 2560 cs 8 / 2 / 4
        // = 25.5 / 19.6 / 18.4 us).
        cs = 1;
        double best = 0.0;
        for (int c = 1; c <= 8; ++c) {
            if (kblocks % c != 0 || (c > 1 && kblocks / c < 2)) continue;
            if (env_fcs >= 1 && c != env_fcs) continue;
            if (a.act_out && env_fcs < 1 && c != 1 && c != 2 && c != 4) continue;
            const int units = mt * c;
            const double eff = (double)units / ((double)((units + wave - 1) / wave) * wave);
            if (eff > best + 0.02) {
                best = eff;
                cs = c;
            }
        }
        splits = cs;
        kb_per = kblocks / cs;
    }
    if (splits / cs > a.max_planes) return 0;
    const uint32_t stage_bytes = (uint32_t)(kBM + bpad) * kBK * 2;
    // ~half the SM's shared memory so two GEMM CTAs co-reside: the next GEMM of
    // the step (PDL) streams its weights while this one drains.
    int stages = std::min(4, (int)(((deep ? kSmemBudget : kSmemBudget / 2) - 1024 - 256) / stage_bytes));
    stages = std::min(stages, std::max(2, kb_per));
    // wide activation tiles (prefill, >= 128 rows): one CTA per SM with a
    // deeper pipeline (EEB_TC_WIDE=1; measured slower on the C2 prefill)
    static const bool wide_stages = std::getenv("EEB_TC_WIDE") && std::atoi(std::getenv("EEB_TC_WIDE")) != 0;
    if (wide_stages && bpad >= 128) stages = std::min(4, (int)((kSmemBudget - 1024 - 256) / stage_bytes));
    if (stages < 2) stages = std::min(8, (int)((kSmemBudget - 1024 - 256) / stage_bytes));
    if (env_stages > 0) stages = std::min(env_stages, (int)((kSmemBudget - 1024 - 256) / stage_bytes));
    if (stages < 2) return 0;
    if (a.head_tri) {
        // measured (gemm_sweep, C2 head 50272 x 2048): 3 stages -> 3 CTAs per SM
        // stream the head at 88% of HBM peak vs 77% with 4 stages / 2 per SM
        static const int env_head_stages = std::getenv("EEB_HEAD_STAGES") ? std::atoi(std::getenv("EEB_HEAD_STAGES")) : 3;
        if (env_head_stages > 0) stages = std::min(env_head_stages, (int)((kSmemBudget - 1024 - 256) / stage_bytes));
    }
    if (a.act_out) {
        static const int env_act_stages = std::getenv("EEB_ACT_STAGES") ? std::atoi(std::getenv("EEB_ACT_STAGES")) : 0;
        if (env_act_stages > 0) stages = std::min(env_act_stages, (int)((kSmemBudget - 1024 - 256) / stage_bytes));
    }
    // smem the epilogue reuses from the drained pipeline stages: the staged
    // [bpad][129] f32 partial (cs > 1) or logits tile (head), plus the head's
    // finished rows when the head is split
    const size_t red_bytes = (size_t)bpad * kRS * 4;
    const size_t need = (cs > 1 || a.head_tri) ? red_bytes * (a.head_tri && cs > 1 ? 2 : 1) : 0;
    while (need > (size_t)stages * stage_bytes && stages < 8) ++stages;
    if (need > (size_t)stages * stage_bytes || 1024 + (size_t)stages * stage_bytes + 256 > (size_t)kSmemBudget) {
        if (a.head_tri || a.act_out) return 0;
        cs = 1;
    }
    int tmem_cols = 32;
    while (tmem_cols < bpad) tmem_cols *= 2;

    TcParams p;
    p.cs = cs;
    p.N = a.N;
    p.K = a.K;
    p.kb_per = kb_per;
    p.kblocks = kblocks;
    p.bpad = bpad;
    p.rh = rh;
    p.stages = stages;
    p.tmem_cols = tmem_cols;
    p.n_active = a.n_active;
    p.part = a.out;
    p.split_stride = a.plane_stride;
    p.head_tri = reinterpret_cast<float4*>(a.head_tri);
    p.act_out = static_cast<__nv_bfloat16*>(a.act_out);
    p.act_kind = a.act_kind;
    p.tiles = tiles;
    p.vocab_off = a.vocab_off;
    // measured slower on C2 (1.654 vs 1.621 ms/step) and far slower where the next
    // GEMM's weights exceed L2 (C4): opt-in with EEB_L2PF=1
    static const bool no_pf = !(std::getenv("EEB_L2PF") && std::atoi(std::getenv("EEB_L2PF")) == 1);
    p.pf = no_pf ? nullptr : static_cast<const char*>(a.pf);
    p.pf_bytes = no_pf || !a.pf ? 0 : a.pf_bytes;
    p.trace = a.trace;
    static const int env_dbg = std::getenv("EEB_GEMM_DBG") ? std::atoi(std::getenv("EEB_GEMM_DBG")) : 0;
    p.dbg = env_dbg;
    static const bool skip_dead = !std::getenv("EEB_SKIP_DEAD") || std::atoi(std::getenv("EEB_SKIP_DEAD")) != 0;
    p.skip_dead = skip_dead ? 1 : 0;
    // measured slower on C2 (1.455 vs 1.412 ms/step: the prefetch stream slows the
    // norm that runs beside it more than the GEMMs gain); opt-in EEB_TC_L2PF=1
    static const int env_l2pf = std::getenv("EEB_TC_L2PF") ? std::atoi(std::getenv("EEB_TC_L2PF")) : 0;
    p.l2pf = env_l2pf;
    const CUtensorMap mw = make_map(a.W, a.N, a.K, kBM);
    const CUtensorMap mx = make_map(a.X, a.max_rows, a.K, bpad);
    // plane output map [planes][max_rows][N] f32, box 128 features x bpad rows
    static const bool env_tma_out = !std::getenv("EEB_TC_TMA_OUT") || std::atoi(std::getenv("EEB_TC_TMA_OUT")) != 0;
    CUtensorMap mo = mw;  // (unused unless tma_out)
    p.tma_out = 0;
    // rows per store chunk: the whole tile when the drained stages hold it,
    // else 32-row multiples, double-buffered when two chunks fit
    const size_t stage_smem = (size_t)stages * stage_bytes;
    int orows = (size_t)bpad * kBM * 4 <= stage_smem ? bpad : (int)(stage_smem / (kBM * 4)) / 32 * 32;
    int obufs = 1;
    if (orows < bpad) {
        const int o2 = (int)(stage_smem / (2 * kBM * 4)) / 32 * 32;
        if (o2 >= 32) {
            orows = o2;
            obufs = 2;
        }
    }
    p.orows = orows;
    p.obufs = obufs;
    if (env_tma_out && !a.head_tri && !a.act_out && cs == 1 && a.out && orows >= 16 &&
        (a.plane_stride * 4) % 16 == 0 && ((size_t)a.N * 4) % 16 == 0) {
        const cuuint64_t dims[3] = {(cuuint64_t)a.N, (cuuint64_t)a.max_rows, (cuuint64_t)(splits / cs)};
        const cuuint64_t strides[2] = {(cuuint64_t)a.N * 4, (cuuint64_t)a.plane_stride * 4};
        const cuuint32_t box[3] = {(cuuint32_t)kBM, (cuuint32_t)orows, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode_fn()(&mo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a.out, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(5, "cuTensorMapEncodeTiled (planes) failed: " + std::to_string((int)r));
        p.tma_out = 1;
    }
    const size_t smem = 1024 + (size_t)stages * stage_bytes + (2 * stages + 1) * 8 + 16;
    p.cs = cs;
    auto kern = cs == 4 ? gemm_tc_kernel<4> : cs == 2 ? gemm_tc_kernel<2> : gemm_tc_kernel<0>;
    EEB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid(mt, splits);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 1;
    attr[1].val.clusterDim.y = cs;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    static const bool force_cl = std::getenv("EEB_TC_CLUSTER_ATTR") != nullptr;
    cfg.numAttrs = cs > 1 || force_cl ? 2 : 1;  // no cluster attribute unless clustering (launch cost)
    p.st = stamp_next(reinterpret_cast<const void*>(kern));
    EEB_CUDA(cudaLaunchKernelEx(&cfg, kern, mw, mx, mo, p));
    return splits / cs;
}

}  // namespace eeb
