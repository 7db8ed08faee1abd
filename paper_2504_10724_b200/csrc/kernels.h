// kernels.h — launch interfaces of the eeb sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace eeb {

// ---- synthetic weights (synth_kernels.cu) ---------------------------------
void synth_linear(int dtype, void* dst, uint64_t seed, int tid, int rows, int cols, float scale,
                  bool zero_signal_rows, int d, cudaStream_t s);
// rows x cols block at (row0, col0) of a [*][full_cols] tensor (a tensor-parallel shard)
void synth_linear_slice(int dtype, void* dst, uint64_t seed, int tid, int rows, int cols, int row0, int col0,
                        int full_cols, float scale, bool zero_signal_rows, int d, cudaStream_t s);
void synth_norm(void* dst_f32, uint64_t seed, int tid, int d, cudaStream_t s);
void synth_embedding(int dtype, void* dst, uint64_t seed, int vocab, int d, cudaStream_t s);
// rows (0 = vocab) vocabulary rows starting at row0 (vocab-parallel shard)
void synth_head(int dtype, void* dst, uint64_t seed, int e, float alpha, int vocab, int d,
                cudaStream_t s, int row0 = 0, int rows = 0);

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

// ---- row kernels (rows.cu) ---------------------------------------------------
// x[i] = emb[tok[i]]; initialises the compact state to the identity.
void launch_embed(int dtype, const void* emb, const int* tok, const int* slot_in, const int* pos_in,
                  int batch, int d, RowState st, cudaStream_t s);
// bf16: embed fused with the first layer's RMSNorm (x = emb[tok], out = norm(x) * g); false if not applicable.
bool launch_embed_norm(int dtype, const void* emb, const int* tok, const int* slot_in, const int* pos_in, int batch,
                       int d, RowState st, float eps, const float* g, void* out, cudaStream_t s);
// x[i] += sum_s part[s][i] (part may be null); out1 = act(x*g1/rms), out2 = act(x*g2/rms) (optional).
// pf / pf_bytes: the next GEMM's weights, prefetched into L2 by the CTAs (optional).
void launch_residual_norm(int dtype, const float* part, int splits, int64_t split_stride, const int* n_active,
                          int max_rows, float* x, int d, float eps, const float* g1, void* out1, const float* g2,
                          void* out2, cudaStream_t s, const void* pf = nullptr, size_t pf_bytes = 0,
                          int min_vec = 1);
// ---- tensor-parallel exchange over peer memory (rows.cu) ---------------------
// Every rank of a TP group owns one exchange buffer ("px") with the same
// layout; `base[p]` is rank p's buffer as mapped in this process (NVLink P2P
// or CUDA IPC; on one device, plain pointers).  Flags are u32 cells written by
// peers with st.release.sys and polled with ld.acquire.sys; each CTA index
// keeps its own epoch counter, and every rank launches the same sequence of
// exchanges with the same grids, so epochs advance in lockstep.
constexpr int kPxMaxRanks = 8;
constexpr int kPxMaxCtas = 1024;    // tp_norm: one CTA per row (prefill chunks <= 1024 rows)
constexpr int kPxGatherCtas = 64;   // head-partial all-gather
struct PxLayout {
    int64_t arrive = 0;   // u32 [kPxMaxRanks][kPxMaxCtas]: rank p's CTA i reached the exchange
    int64_t pushed = 0;   // u32 [kPxMaxRanks][kPxMaxCtas]: rank p's reduced slice of row i has landed here
    int64_t epoch = 0;    // u32 [kPxMaxCtas]: this rank's per-CTA epoch counters (local only)
    int64_t g_arrive = 0; // u32 [kPxMaxRanks][kPxGatherCtas]
    int64_t g_epoch = 0;  // u32 [kPxGatherCtas]
    int64_t planes = 0;   // f32 row-parallel GEMM partial planes (this rank's)
    int64_t red = 0;      // f32 [rows][d]: reduced rows (each rank pushes its 1/N slice)
    int64_t head = 0;     // f32 this rank's exit-head tile partials (vocab shard)
    int64_t planes_elems = 0, rows = 0, head_elems = 0, bytes = 0;
};
struct PxPeers {
    char* base[kPxMaxRanks];
    int nranks = 0, rank = 0;
    PxLayout lay;
};
// Two-shot all-reduce of the row-parallel partials fused with the residual add
// and RMSNorm: CTA i of rank r sums the r-th 1/N slice of row i over every
// rank's `planes` planes (rank-major, plane-minor: the order of the all-shards
// context's split-K reduction) and pushes it to every rank (reduce-scatter +
// all-gather); every rank then applies x += sum, out1 = T(rmsnorm(x) g1),
// out2 likewise — so all ranks hold bit-identical residual streams.
void launch_tp_norm(int dtype, const PxPeers& px, int planes, int64_t plane_stride, const int* n_active, int max_rows,
                    float* x, int d, float eps, const float* g1, void* out1, const float* g2, void* out2,
                    cudaStream_t s, int min_vec = 1);
// All-gather of the vocab-parallel exit-head partials: rank p's `region`
// floats (its px head area) land at dst + p * region on every rank.
void launch_px_gather(const PxPeers& px, int64_t region, float* dst, cudaStream_t s);

// out[i][:] = sum_s part[s][i][:] for the live rows (tensor-parallel partial before all-reduce).
void launch_plane_sum(const float* part, int splits, int64_t split_stride, const int* n_active, int max_rows, int d,
                      float* out, int num_sms, cudaStream_t s);
// out[i][n] = relu(sum_s part) or silu(gate)*up over interleaved (gate, up) columns.
void launch_act(int dtype, const float* part, int splits, int64_t split_stride, const int* n_active, int max_rows,
                int N, bool swiglu, void* out, int num_sms, cudaStream_t s);

// ---- decode GEMM (gemm_cc.cu: CUDA cores; gemm_tc.cu: tcgen05) ---------------
// y[b][n] = sum_k X[b][k] * W[n][k], written as split-K partial planes:
// plane s at out + s * plane_stride, row stride N.  Consumers reduce the
// planes in a fixed order (deterministic, no atomics).
struct GemmArgs {
    int dtype;          // weight / activation dtype
    const void* W;      // [N, K] row-major (K contiguous)
    const void* X;      // [max_rows, K] activations, row-major
    const int* n_active;
    int max_rows;
    int N, K;
    float* out;         // partial planes
    int64_t plane_stride;
    int max_planes;
    int num_sms;
    // Exit-head epilogue (tier 2 only): instead of logits, write per (row, 128-
    // vocab tile) partials {max, sum exp(l - max), argmax} to head_tri[row *
    // tiles + tile] (float4, argmax as int bits); decide merges them.
    float* head_tri = nullptr;
    int vocab_off = 0;
    // Fused MLP activation (tier 2 only): write act(y) as bf16 [rows][N] (ReLU,
    // act_kind 1) or [rows][N/2] (SwiGLU over interleaved gate/up, act_kind 2).
    void* act_out = nullptr;
    int act_kind = 0;  // global id of this shard's first vocabulary row (vocab-parallel heads)
    // L2 prefetch of the NEXT GEMM's weights (tier 2): issued by this GEMM's
    // CTAs right after their own first weight tiles, so the HBM stream stays
    // busy through this GEMM's tail and the non-GEMM kernels in between.
    const void* pf = nullptr;
    size_t pf_bytes = 0;
    unsigned long long* trace = nullptr;  // timing experiments (tier 2): 8 stamps per CTA
};
// Tier 1: CUDA cores (any dtype, <= 64 rows).  Returns the planes written.
int gemm_cc(const GemmArgs& a, cudaStream_t s);
// Tier 2: tcgen05 + TMA (bf16, 16..256 rows).  Returns planes, 0 if not applicable.
int gemm_tc(const GemmArgs& a, cudaStream_t s);
bool gemm_tc_available();
int tc_min_rows();
// 2-D TMA map over a row-major bf16 [rows][cols] matrix, box {64 cols, box_rows},
// 128-byte swizzle (the K-major UMMA operand layout).  out_map: 128 B.
void make_bf16_map(void* out_map, const void* ptr, int rows, int cols, int box_rows);
// 3-D TMA map over one layer's bf16 KV cache [slots*Hkv][max_seq][head_dim],
// box {64 dims, box_rows positions, 1}, 128-byte swizzle.  out_map: 128 B.
void make_kv_tensor_map(void* out_map, const void* base, int head_dim, int max_seq, int slots_x_heads,
                        int box_rows);

// ---- attention (attention.cu) ------------------------------------------------
struct AttnArgs {
    int dtype;
    const float* qkv;        // partial planes of the QKV GEMM, rows of dq + 2 dkv
    int splits;
    int64_t split_stride;
    void* k_cache;           // this layer: [pages][Hkv][page_size][hd] (unpaged: page = slot, page_size = S)
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
    const void* k_map;       // bf16: TMA maps of this layer's K / V (128 B each), else null
    const void* v_map;
    const void* k_map8 = nullptr;  // the same tensors with 8-row boxes (exact tails)
    const void* v_map8 = nullptr;
    int num_sms;
    int kv_ready = 0;        // prefill: every row's K/V is already in the cache (launch_kv_append)
    // Paged KV pool: position p of slot s lives in page page_table[s * pages_per_seq + p / page_size]
    // at row p % page_size.  Unpaged: page_size = max_seq, pages_per_seq = 1, table = identity.
    const int* page_table = nullptr;
    int page_size = 0;
    int pages_per_seq = 1;
    // Prefill (kv_ready): query blocks of <= 64 consecutive rows of one
    // sequence, {first row, rows, slot, position of the first row}; the
    // tensor-core prefill kernel runs one CTA per (block, query head).
    const int4* pf_items = nullptr;
    const int* pf_n_items = nullptr;
    int pf_max_items = 0;
    // Decode KV split (flash-decoding): kv_splits CTAs share a (row, kv head),
    // each over a contiguous range of 64-position chunks; partials
    // {O (unnormalised), max, sum} go to kv_part and the last split to finish
    // (kv_ticket, zero between launches) combines them in split order.
    int kv_splits = 1;
    float* kv_part = nullptr;   // [max_rows][Hkv][kv_splits][8][hd + 2]
    int* kv_ticket = nullptr;   // [max_rows][Hkv]
    int dbg = 0;                // timing experiments (attention_dec, EEB_ATTN_DBG): 1 no compute, 2 no K/V loads
    int pre_stages = 1;         // attention_dec: ring stages issued before the prologue (EEB_ATTN_PRE)
    const void* pf = nullptr;   // the O GEMM's weights, prefetched into L2 during the attention (optional)
    size_t pf_bytes = 0;
};
// Device address of (page-table row of slot, position, kv head, dim 0) in a layer's K or V cache.
__host__ __device__ inline int64_t kv_elem_offset(const AttnArgs& a, int slot, int pos, int g) {
    const int pg = a.page_table[(int64_t)slot * a.pages_per_seq + pos / a.page_size];
    return (((int64_t)pg * a.n_kv_heads + g) * a.page_size + pos % a.page_size) * a.head_dim;
}
void launch_attention(const AttnArgs& a, cudaStream_t s);
// Streaming decode attention (attention_dec.cu): bf16, head_dim 64, decode
// (not kv_ready), no KV split.  Returns false where it does not apply.
bool launch_attention_dec(const AttnArgs& a, cudaStream_t s);
// Prefill: RoPE the keys and write K/V of every live row into the cache
// (a chunk's rows attend to each other, so the append precedes the attention).
void launch_kv_append(const AttnArgs& a, cudaStream_t s);
// Prefill: kv_depth[slot[i]][pos[i]] = depth for the rows of the chunk.
void launch_mark_depth(int rows, const int* slot, const int* pos, uint8_t* kv_depth, int max_seq, int depth,
                       cudaStream_t s);

// ---- exit head, decisions, compaction, histogram (exit_head.cu) ------------
struct HeadOut {             // result of one head on the live rows (compact-indexed)
    int* tok;
    float* conf;
    float* logp;
};
// Head logits arrive as split-K planes; logits_out (optional) receives the sum.
void launch_head_reduce(const float* part, int splits, int64_t split_stride, int vocab, const int* n_active,
                        int max_rows, HeadOut h, float* logits_out, cudaStream_t s);

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
    const float* head_tri = nullptr;  // optional: per-(row, tile) partials from the fused head GEMM (merged here)
    int head_tiles = 0;               // tiles per shard region
    int head_shards = 1;              // regions (tensor-parallel ranks)
    int64_t head_shard_stride = 0;    // float4 entries between regions
    StepOutDev out;
    int layers[64];          // exit ladder (profile mode maps head index -> layer)
    // Captured introspective step: the rest of the step (deeper layers and
    // heads) is a conditional graph body run only if a row survives this head
    // (decide sets the condition from the survivor count).
    int has_cond = 0;
    cudaGraphConditionalHandle cond = 0;
    // fused-head merge spread over CTAs (a warp per row); the last CTA to
    // finish, counted here (zero between launches), decides and compacts
    int* ticket = nullptr;
};
void launch_decide(const DecideArgs& a, cudaStream_t s);
// x_nxt[j] = x_cur[src[j]] (and the normalised row h) for live rows of the compacted state.
void launch_gather_rows(const float* x_cur, float* x_nxt, const void* h_cur, void* h_nxt, int h_bytes_per_row,
                        const int* src, const int* n_active, int max_rows, int d, cudaStream_t s);
// Histogram (K4), breach count and fixed-order logprob sum over `batch` rows;
// records each row's computed depth in the KV depth map (its exit layer, or
// computed_depth when > 0: the profiling pass runs every row to full depth).
void launch_finalize(int batch, int n_exits, StepOutDev out, const int* slot_in, const int* pos_in,
                     uint8_t* kv_depth, int max_seq, int computed_depth, cudaStream_t s);

}  // namespace eeb
