// kernels.h — launch interfaces of the eeb sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace eeb {

// ---- synthetic weights (synth_kernels.cu) ---------------------------------
void synth_linear(int dtype, void* dst, uint64_t seed, int tid, int rows, int cols, float scale,
                  bool zero_signal_rows, int d, cudaStream_t s);
void synth_norm(void* dst_f32, uint64_t seed, int tid, int d, cudaStream_t s);
void synth_embedding(int dtype, void* dst, uint64_t seed, int vocab, int d, cudaStream_t s);
void synth_head(int dtype, void* dst, uint64_t seed, int e, float alpha, int vocab, int d,
                cudaStream_t s);

// ---- per-step row state ----------------------------------------------------
// Rows are kept compact: entries [0, *n_active) are live.  row_of maps a
// compact index to the caller's row (the output index).
struct RowState {
    int* n_active;   // [1]
    int* row_of;     // [maxB]
    int* slot;       // [maxB]
    int* pos;        // [maxB]
    float* x;        // [maxB, d] residual stream (f32)
};

// ---- elementwise / normalisation (rows.cu) ---------------------------------
// x[i] = emb[tok[i]]; initialises the compact state to the identity.
void launch_embed(int dtype, const void* emb, const int* tok, const int* slot_in, const int* pos_in,
                  int batch, int d, RowState st, cudaStream_t s);
// out[i] = act(x[i] * gain / rms(x[i])) for live rows.
void launch_rmsnorm(int dtype, const float* x, const float* gain, const int* n_active, int max_rows,
                    int d, float eps, void* out, cudaStream_t s);

// ---- GEMM (gemm_cc.cu: CUDA-core split-K; gemm_tc.cu: tcgen05) -------------
enum EpilogueMode : int {
    kStoreF32 = 0,   // out_f32[i][n] = y
    kResidAdd = 1,   // x[i][n] += y
    kReluAct = 2,    // out_act[i][n] = relu(y)
    kSwigluAct = 3,  // out_act[i][j] = silu(y[2j]) * y[2j+1]
};
struct GemmArgs {
    int dtype;          // weight / activation dtype
    const void* W;      // [N, K] row-major (K contiguous)
    const void* X;      // [maxB, K] activations, row-major
    const int* n_active;
    int max_rows;       // capacity / launch bound for rows
    int N, K;
    int mode;
    float* out_f32;     // kStoreF32 / kResidAdd target, row stride ldo
    void* out_act;      // kReluAct / kSwigluAct target
    int ldo;
    float* workspace;   // split-K partials
    int64_t workspace_elems;
    int num_sms;
};
// Tier 1: CUDA cores (any dtype, any batch).
void gemm_cc(const GemmArgs& a, cudaStream_t s);
// Tier 2: tcgen05 + TMA (bf16, batch >= 16).  Returns the number of kernels
// launched, 0 when the shape is not applicable (caller falls back to tier 1).
int gemm_tc(const GemmArgs& a, cudaStream_t s);
bool gemm_tc_available();

// ---- attention (attention.cu) ------------------------------------------------
struct AttnArgs {
    int dtype;
    const float* qkv;        // [maxB, dq + 2 dkv] f32
    void* k_cache;           // this layer: [slots][Hkv][S][hd]
    void* v_cache;
    const uint8_t* kv_depth; // [slots][S] layers computed per position
    const float* rope_cos;   // [S][hd/2]
    const float* rope_sin;
    const int* n_active;
    const int* slot;
    const int* pos;
    int max_rows;
    int layer;               // 1-indexed
    int n_heads, n_kv_heads, head_dim, max_seq;
    void* out;               // [maxB, dq] act dtype
};
void launch_attention(const AttnArgs& a, cudaStream_t s);

// ---- exit head, decisions, compaction, histogram (exit_head.cu) ------------
struct HeadOut {             // result of one head on the live rows (compact-indexed)
    int* tok;
    float* conf;
    float* logp;
};
void launch_head_reduce(const float* logits, int vocab, const int* n_active, int max_rows,
                        HeadOut h, cudaStream_t s);

struct StepOutDev {          // caller-row-indexed outputs (device)
    int32_t* exit_layer;
    int32_t* token_id;
    float* confidence;
    float* logprob;
    uint8_t* breached;
    uint8_t* unchanged;
    int32_t* bin;            // exit-head index used (histogram bin)
    int64_t* hist;           // [n_exits]
    int64_t* n_breached;
    double* sum_logprob;
    int32_t* head_token;     // [B][n_exits] (profile)
    float* head_confidence;
    float* head_logprob;
};

struct DecideArgs {
    int policy;              // eeb_token_policy
    int exit_index;          // head just evaluated
    int n_exits;
    int exit_layer;          // layer of that head
    int num_layers;
    int serving_depth;
    int is_final;            // last head evaluated in this step
    float th;
    int max_rows;
    RowState cur;            // state the head ran on
    RowState nxt;            // compaction target (introspective, non-final)
    int* gather_src;         // [maxB] nxt index -> cur index
    HeadOut head;
    StepOutDev out;
    int layers[64];          // exit ladder (profile mode maps head index -> layer)
};
void launch_decide(const DecideArgs& a, cudaStream_t s);
// x_nxt[j] = x_cur[src[j]] for live rows of the compacted state.
void launch_gather_rows(const float* x_cur, float* x_nxt, const int* src, const int* n_active,
                        int max_rows, int d, cudaStream_t s);
// Histogram (K4), breach count and fixed-order logprob sum over `batch` rows;
// records each row's computed depth in the KV depth map.
void launch_finalize(int batch, int n_exits, StepOutDev out, const int* slot_in, const int* pos_in,
                     uint8_t* kv_depth, int max_seq, cudaStream_t s);

}  // namespace eeb
