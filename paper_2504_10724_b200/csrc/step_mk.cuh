// step_mk.cuh — host/device interface of the persistent decode-step kernel.
//
// The whole batched early-exit decode step (the batched form
// of Simulator::serve_one's token loop, engine.hpp:344-386) runs as ONE
// cooperative launch with one CTA per SM.  The host compiles the step into a
// program of phases (GEMM, residual+RMSNorm, attention, activation, exit-head
// reduction, exit decision, finalize) kept in shared memory; every CTA walks
// the same program, phases separated by grid-wide barriers.  Weights never
// depend on the step's data, so the TMA producer warp streams every GEMM
// phase's weight tiles into the shared-memory ring without waiting for those
// barriers: the weight stream runs across phase boundaries, which a chain of
// separate kernel launches cannot do.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "kernels.h"

namespace eeb {
namespace mk {

constexpr int kThreads = 256;  // 8 warps: W producer, MMA, control/X producer, SIMT, 4 x epilogue
constexpr int kSimtWarps = 6;  // warps 2..7 run the non-GEMM phases
constexpr int kBM = 128;       // UMMA M: output features per tile
constexpr int kBK = 64;        // k-block: one 128-byte swizzle atom of bf16
constexpr int kMaxSeg = 8;     // partial-sum segments one CTA may own in a GEMM phase
constexpr int kMaxRows = 128;  // rows per step on this path (UMMA N <= 128, live list in smem)
constexpr int kSegUnroll = 10; // partial segments of one tile summed with all loads in flight
constexpr int kHeadChunk = 16; // vocabulary tiles (x128) per exit-head reduction task
constexpr int kAttnScratchBytes = (8 * 64 + 128) * 4;  // per SIMT warp attention scratch (q, k, v), in the X ring

enum PhaseKind : int {
    kPhaseGemm = 0,        // y = X W^T, stream-K, partial sums -> partial buffer
    kPhaseNorm = 1,        // x (+)= sum(partials of src); out = bf16(rmsnorm(x) * gain)  (embed: x = emb[tok])
    kPhaseAttn = 2,        // q,k,v = sum(partials of src); RoPE; KV append; attention -> attn
    kPhaseAct = 3,         // hmid = act(sum(partials of src))
    kPhaseHeadReduce = 4,  // per row: max / argmax / sum-exp over the vocabulary -> stats
    kPhaseDecide = 5,      // exit rule, outputs, survivor compaction (every CTA, identical)
    kPhaseFinalize = 6,    // histogram, breach count, logprob sum, KV depth map (CTA 0)
};

enum PhaseFlag : int {
    kFlagEmbed = 1,    // norm: x = emb[tok] instead of x += partials
    kFlagOutHead = 2,  // norm: write the exit-head input buffer (hh) instead of h
    kFlagFinal = 4,    // decide: last head evaluated in this step
};

struct Phase {
    int kind;
    int layer;       // 1-based layer (gains, KV cache)
    int exit_index;  // head index (decide / head reduce)
    int src;         // GEMM phase whose partials are consumed (-1 none)
    int wmap, xmap;  // tensor-map table indices (weights [N][K], activations [rows][K])
    int N, K, kb, tiles, total;
    int flags;
    int gain;        // index into the gains table
    int exit_layer;  // decide: layer of the head
    int pad[2];
};

struct Params {
    const Phase* phases;
    int n_phases;
    const CUtensorMap* maps;
    float* partials;  // [G][kMaxSeg][bpad][128]
    unsigned* bar;    // grid barrier state (u64 arrival counter at +8 bytes)
    unsigned long long bar_base;  // arrivals before this launch (host-tracked, stream-ordered)
    int batch;        // rows in this step
    int bpad;         // UMMA N: rows padded to 16
    int w_stages, x_stages;
    int bar_mode, dbg, l2_ahead;  // bar_mode 0: counter barrier; dbg / l2_ahead: timing experiments
    unsigned long long* trace;    // optional [G][n_phases][8] globaltimer stamps
    const void* const* wbase;     // timing experiments only
    int n_segtab;                 // entries of the segment table (copied to shared memory)
    // model
    int D, F, dq, dkv, H, Hkv, hd, V, S, L, n_exits, mlp_kind, policy, serving_depth;
    float eps, th;
    const __nv_bfloat16* emb;   // [V][D]
    const float* const* gains;  // attn_norm[L], mlp_norm[L], head_norm[E]
    __nv_bfloat16* k_cache;     // [L][slots][Hkv][S][hd]
    __nv_bfloat16* v_cache;
    long long kv_layer_elems;
    uint8_t* kv_depth;          // [slots][S]
    const float* rope_cos;      // [S][hd/2]
    const float* rope_sin;
    // step io (device)
    const int* tok;
    const int* slot;
    const int* pos;
    float* x;             // [batch][D] residual stream, caller-row indexed
    __nv_bfloat16* h;     // [bpad][D]  compact rows
    __nv_bfloat16* hh;    // [bpad][D]
    __nv_bfloat16* attn;  // [bpad][dq]
    __nv_bfloat16* hmid;  // [bpad][F]
    float4* stats;        // [bpad][n_chunks] per vocabulary chunk {max, sum-exp, argmax bits, -}
    StepOutDev out;
    int exit_layers[64];
};

// Shared-memory bytes for a configuration (host and device agree).
__host__ __device__ inline unsigned smem_bytes(int bpad, int w_stages, int x_stages, int n_phases, int n_segtab) {
    return 1024u + (unsigned)w_stages * (kBM * kBK * 2) + (unsigned)x_stages * (unsigned)(bpad * kBK * 2) +
           (unsigned)(2 * w_stages + 2 * x_stages + 8) * 8u + 64u + (unsigned)n_phases * (unsigned)sizeof(Phase) +
           (unsigned)(kMaxRows + 64) * 4u + 256u + (unsigned)n_segtab * 16u + 16u + 6u * 40u;
}

// Launch the program (cooperative, grid = SM count).  segtab: per GEMM phase
// and output tile {first CTA, its partial slot, segment count} (Phase::pad[0]
// is the phase's offset into it).
void launch(const Params& p, const int4* segtab, int grid, cudaStream_t s);

}  // namespace mk
}  // namespace eeb
