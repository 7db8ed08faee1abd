/*
 * eeb.h — C ABI of the B200-native batched early-exit (EE) decode step.
 *
 * This is the drop-in seam for the reference's decode step.  In the reference
 * (HELIOS simulator, /root/reference/proj/include/eeserve/) `Simulator::serve_one`
 * obtains each token's exit-head verdicts from a pre-computed trace
 * (`tok.for_model(model)`, engine.hpp:345) and then applies the token policy
 * (engine.hpp:349-366).  `eeb_decode_step` replaces exactly that pair for a
 * whole batch: it runs the real decoder layers on the GPU, evaluates the exit
 * heads, applies the same exit rule and returns, per row, the `ExitObservation`
 * fields (trace.hpp:17-22) plus the breached / unchanged flags
 * (engine.hpp:353,358,363,366) and the exit-layer histogram that feeds the
 * profiler (`ExitHistogram`, pht.hpp:15-38; `record_token`, pht.hpp:92-102).
 *
 * Conventions (mirroring the reference):
 *   - status codes map 1:1 onto the reference's exception types
 *     (errors.hpp:9-30); no C++ exception crosses this boundary;
 *   - one context per (host thread, GPU); calls on a context are externally
 *     serialised; distinct contexts are independent (the reference's
 *     `sweep -j` model, eeserve.cpp:220-259);
 *   - the caller owns every buffer passed in; model descriptors are copied.
 *
 * Plain C: no torch or CUDA types in any signature (streams are opaque).
 */
#ifndef EEB_H_
#define EEB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EEB_ABI_VERSION 1

/* ↔ errors.hpp:9-30 (ValidationError, CapacityError, DomainError, StalenessError). */
typedef enum {
    EEB_OK = 0,
    EEB_E_VALIDATION = 1,
    EEB_E_CAPACITY = 2,
    EEB_E_DOMAIN = 3,
    EEB_E_STALE = 4,
    EEB_E_CUDA = 5
} eeb_status;

/* ↔ Simulator::TokenPolicy (engine.hpp:156) plus the profiling pass of
 * run_eval_cycle (engine.hpp:261-263, every head observed at full depth). */
typedef enum {
    EEB_FLAT = 0,          /* helios serving: every row runs `serving_depth` layers (trace.hpp:86-97) */
    EEB_INTROSPECTIVE = 1, /* earliest confident head exits (trace.hpp:69-76); survivors compacted   */
    EEB_FULL_DEPTH = 2,    /* vanilla: final head only, breached = false (engine.hpp:360-364)       */
    EEB_PROFILE = 3        /* all heads on all rows at full depth: a full ModelTokenRecord per row  */
} eeb_token_policy;

typedef enum { EEB_F32 = 0, EEB_BF16 = 1 } eeb_dtype;
typedef enum { EEB_MLP_RELU = 0, EEB_MLP_SWIGLU = 1 } eeb_mlp_kind;

/* Model/layer descriptor ↔ ModelSpec (model_spec.hpp:15-37), extended
 * additively with the real architecture dimensions the reference lacks. */
typedef struct {
    int32_t num_layers;
    int32_t d_model;
    int32_t n_heads;
    int32_t n_kv_heads;
    int32_t d_ffn;
    int32_t vocab;
    int32_t n_exits;
    const int32_t* exit_layers;   /* strictly increasing, last == num_layers (model_spec.hpp:62-83) */
    const float* exit_coverage;   /* biased-head calibration: fraction of tokens whose earliest
                                     confident head (at design_th) is <= each exit; NULL = defaults */
    float design_th;              /* threshold the exit heads are calibrated for (policy.hpp:51) */
    int32_t dtype;                /* eeb_dtype of weights / GEMM activations / KV */
    int32_t mlp_kind;             /* eeb_mlp_kind */
    int32_t max_slots;            /* KV slot pool (memory_model.hpp:58-72 sizes it) */
    int32_t max_seq_len;          /* KV positions per slot */
    uint64_t seed;                /* weights are a pure function of (seed, tensor, index) */
    float rope_theta;
    float norm_eps;
    /* Tensor parallelism (C5: 70B over 8 GPUs): 0/1 = none.  tp_rank >= 0: this
     * context holds shard tp_rank (its q/kv heads, d_ffn/tp MLP columns,
     * vocab/tp head rows) and sums row-parallel partials / gathers head
     * partials over the context's NCCL communicator (eeb_nccl_init).
     * tp_rank = -1: all tp shards in this context, combined locally. */
    int32_t tp_size;
    int32_t tp_rank;
} eeb_model_desc;

/* Per-step outputs, all arrays of length `batch` unless noted.  Any pointer
 * may be NULL (not returned).  Row order = input row order. */
typedef struct {
    int32_t* exit_layer;     /* layer the row's token left the network at           */
    int32_t* token_id;       /* argmax of the exit head used (trace.hpp:19)         */
    float* confidence;       /* max softmax probability               */
    float* logprob;          /* log-prob of the emitted token at that head          */
    uint8_t* breached;       /* confidence < th (engine.hpp:353,358); 0 for full depth */
    uint8_t* unchanged;      /* 1/0 = head token ==/!= final token; 2 = unknown (final head not run) */
    int64_t* hist;           /* [n_exits] step exit histogram (K4)                  */
    int64_t* n_breached;     /* [1] breached rows in this step                      */
    double* sum_logprob;     /* [1] sum of logprob over rows, fixed order (fp64)    */
    /* EEB_PROFILE only: every head's observation, [batch][n_exits] row-major. */
    int32_t* head_token;
    float* head_confidence;
    float* head_logprob;
} eeb_step_out;

typedef struct eeb_ctx eeb_ctx;

/* Lifecycle. */
eeb_status eeb_create(int device, eeb_ctx** out);
void eeb_destroy(eeb_ctx* ctx);
const char* eeb_last_error(void);   /* thread-local message of the last failure */
int eeb_abi_version(void);

/* Register a model (descriptor copied) and allocate its KV slot pool.
 * No weights are resident until eeb_load_layers. */
eeb_status eeb_model_register(eeb_ctx* ctx, const eeb_model_desc* desc, int* model);

/* Greedy layer loader ↔ do_load (engine.hpp:197-216) / apply_load
 * (memory_model.hpp:86-105): make layers [1, to_depth] plus the base weights
 * (embedding, exit heads) resident.  Weights are materialised on device from
 * the model seed.  Shrinking frees layers deeper than to_depth. */
eeb_status eeb_load_layers(eeb_ctx* ctx, int model, int to_depth);
eeb_status eeb_evict(eeb_ctx* ctx, int model);   /* ↔ evict_model (memory_model.hpp:104) */
eeb_status eeb_loaded_depth(eeb_ctx* ctx, int model, int* depth);

/* Caller-supplied weights (real checkpoints; tp_size == 1 models).  The packed
 * host layout, all tensors row-major with K contiguous, in the model dtype
 * except the norm gains (f32), each part at a 256-byte aligned offset:
 *   layer l:  0 attn_norm [D] f32 | 1 mlp_norm [D] f32 | 2 Wqkv [dq + 2 dkv][D]
 *             (q rows, k rows, v rows) | 3 Wo [D][dq] | 4 Wup [F][D] (ReLU) or
 *             [2F][D] (SwiGLU: gate and up rows interleaved) | 5 Wdown [D][F]
 *   base:     embedding [V][D] | exit heads e = 0..n_exits-1 [V][D] | head
 *             norm gains e = 0..n_exits-1 [D] f32
 * Replaces the reference's `do_load` source (engine.hpp:197-216: a model's
 * layers in CPU memory moved to the GPU); SURVEY §8(b) eeb_load_layers(ctx,
 * model, from, to, pinned_host, bytes). */
typedef struct {
    int64_t layer_bytes, base_bytes;  /* bytes of one packed layer / of the base weights */
    int64_t layer_off[6];             /* part offsets inside a layer */
    int64_t base_off[1 + 2 * 64];     /* embedding, heads, head norms (-1 past n_exits) */
} eeb_weight_layout_t;
eeb_status eeb_weight_layout(eeb_ctx* ctx, int model, eeb_weight_layout_t* out);
/* Copy one packed layer (1-based) / the base weights into the host tier (pinned;
 * the source of eeb_load_layers and eeb_load_layers_async from then on).  The
 * tier is a prefix: layer l needs layers < l staged.  A resident layer's device
 * copy is refreshed. */
eeb_status eeb_host_stage_layer(eeb_ctx* ctx, int model, int layer, const void* host, int64_t bytes);
eeb_status eeb_host_stage_base(eeb_ctx* ctx, int model, const void* host, int64_t bytes);
/* Layers [from, to] from one buffer of (to - from + 1) packed layers: staged to
 * the host tier and made resident (from <= loaded_depth + 1); returns when done. */
eeb_status eeb_load_layers_from(eeb_ctx* ctx, int model, int from, int to, const void* host, int64_t bytes);

/* Reserve device memory for a later load of layers up to `depth` (and the
 * base weights): the buffers are allocated and parked in the context's weight
 * block pool, so loads and reloads while serving (model switches, depth
 * changes) reuse them instead of calling cudaMalloc / cudaFree (host time,
 * device synchronisation).  Pooled blocks go back to the driver when any
 * allocation of the library fails. */
eeb_status eeb_weight_reserve(eeb_ctx* ctx, int model, int depth);

/* Host tier ↔ the model held in CPU memory that HELIOS's greedy loader pulls
 * layers from (engine.hpp:197-216; memory_model.hpp:76-105): layers [1, depth]
 * plus the base weights (embedding, exit heads) packed into pinned host
 * memory, one blob per layer.  Blocking. */
eeb_status eeb_host_stage(eeb_ctx* ctx, int model, int depth);
/* Asynchronous greedy load ↔ do_load (engine.hpp:197-216) with a real
 * transfer instead of the modelled bytes / 8.4 GB/s: layers (loaded, to_depth]
 * (and the base weights on the first load) are copied from the host tier by
 * pinned cudaMemcpyAsync on the context's load stream, one event per layer.
 * Returns immediately; decode steps that need only already-resident layers
 * (flat at the old depth) run concurrently, a step that needs an in-flight
 * layer waits on its event on the device (no host block).  to_depth <= loaded
 * shrinks synchronously like eeb_load_layers.  EEB_E_CAPACITY if the host tier
 * does not hold the layers. */
eeb_status eeb_load_layers_async(eeb_ctx* ctx, int model, int to_depth);
/* Block until the model's async load has landed; seconds = its measured
 * duration on the load stream (CUDA events), bytes = bytes copied — the
 * stall do_load charges to the next TTFT (engine.hpp:205-216). */
eeb_status eeb_load_wait(eeb_ctx* ctx, int model, double* seconds, int64_t* bytes);
eeb_status eeb_weight_bytes(eeb_ctx* ctx, int model, int depth, int64_t* bytes);

/* Clear the KV of slots (positions marked as never computed). */
eeb_status eeb_reset_slots(eeb_ctx* ctx, int model, int32_t n, const int32_t* slot_ids);

/* Paged KV pool (replaces the slot-contiguous pool sized by
 * kv_bytes_per_slot x max_batch, memory_model.hpp:53-72).  configure_pages
 * re-creates the model's pool as n_pages pages of page_size positions
 * (multiple of 64, at most 64 pages per sequence) — call it before the first
 * step; it drops every slot's KV.  A slot takes pages from a free list as its
 * positions grow: eeb_decode_step / eeb_prefill (host arrays) reserve them
 * themselves, eeb_decode_step_device needs eeb_kv_reserve first (its positions
 * are device-side).  Out of pages -> EEB_E_CAPACITY (CapacityError).
 * eeb_kv_release returns a finished request's pages (continuous batching:
 * the slot is free for the next request).  bf16 models with head_dim 64/80/128. */
eeb_status eeb_kv_configure_pages(eeb_ctx* ctx, int model, int32_t page_size, int32_t n_pages);
eeb_status eeb_kv_reserve(eeb_ctx* ctx, int model, int32_t slot, int32_t n_positions);
eeb_status eeb_kv_release(eeb_ctx* ctx, int model, int32_t slot);
eeb_status eeb_kv_pages(eeb_ctx* ctx, int model, int32_t* page_size, int32_t* n_pages, int32_t* n_free);

/* The decode step ↔ Simulator::serve_one token loop (engine.hpp:344-386),
 * batched per SPEC.md:465-473.  Row i decodes `input_tokens[i]` at position
 * `positions[i]` of KV slot `slot_ids[i]`.
 *   flat:          head at the deepest exit <= serving_depth; exit_layer = serving_depth
 *   introspective: shallowest head with confidence >= th, final head forced
 *   full_depth:    final head; exit_layer = num_layers, breached = 0
 *   profile:       every head on every row (introspective rule picks exit_layer)
 * Host-pointer variant: inputs/outputs are host memory (pageable or pinned);
 * the H2D/D2H copies are part of the call, which returns when `out` is filled. */
eeb_status eeb_decode_step(eeb_ctx* ctx, int model, int serving_depth, int policy, float th,
                           int32_t batch, const int32_t* slot_ids, const int32_t* input_tokens,
                           const int32_t* positions, eeb_step_out* out);

/* Device-resident variant: every pointer (inputs and outputs) is device
 * memory; the call is asynchronous on the context stream (eeb_synchronize). */
eeb_status eeb_decode_step_device(eeb_ctx* ctx, int model, int serving_depth, int policy, float th,
                                  int32_t batch, const int32_t* d_slot_ids,
                                  const int32_t* d_input_tokens, const int32_t* d_positions,
                                  eeb_step_out* d_out);
eeb_status eeb_synchronize(eeb_ctx* ctx);

/* Prefill ↔ the prefill phase of Simulator::serve_one (engine.hpp:333-341:
 * prompt_len x depth layer-token passes, charged to TTFT), batched.  The
 * prompts of n_seq sequences — tokens concatenated in sequence order, lens[k]
 * tokens for sequence k starting at position start_pos[k] of KV slot
 * slot_ids[k] — run through layers 1..depth, writing their K/V at every
 * layer <= depth and marking those positions computed to `depth` (deeper
 * layers mask them, as for a token that exited at `depth`).  Chunked into
 * passes of <= 256 tokens (one pass over the loaded layers per chunk; a later
 * chunk attends to the KV of earlier ones).  No token is emitted: the first
 * output token comes from the decode step, as in serve_one's token loop.
 * start_pos > 0 re-prefills a suffix (after load-more / switch, SPEC re-prefill).
 * Host pointers; the call returns when the KV is written.  SURVEY §8(b) sketch:
 * eeb_prefill(ctx, model, depth, slot, prompt, len). */
eeb_status eeb_prefill(eeb_ctx* ctx, int model, int depth, int32_t n_seq, const int32_t* slot_ids,
                       const int32_t* start_pos, const int32_t* lens, const int32_t* tokens);

/* Capture the step for (model, depth, policy, batch) into a CUDA graph and
 * reuse it on later identical calls (0 = off, 1 = on; default on). */
eeb_status eeb_set_graphs(eeb_ctx* ctx, int enable);

/* Kernel tier override for tests: 0 = auto (tcgen05 GEMMs for bf16 models,
 * CUDA-core GEMV for f32), 1 = CUDA-core GEMV only, 2 = tcgen05 GEMMs
 * (EEB_E_DOMAIN where not applicable). */
eeb_status eeb_set_gemm_tier(eeb_ctx* ctx, int tier);

/* In-graph launch timeline (diagnostics; the bench's roofline source).
 * max_launches > 0: every later decode step records, per kernel launch, the
 * first CTA start and the last warp exit (%globaltimer, written by the kernels
 * themselves inside the captured PDL graph); 0 turns it off.  Toggling drops
 * the captured graphs. */
eeb_status eeb_debug_stamps(eeb_ctx* ctx, int max_launches);
/* JSON {"launches": [{"kernel", "start_ns", "end_ns", "ctas"}, ...]} of the
 * last decode step, in launch order, times relative to its first CTA start. */
eeb_status eeb_debug_stamps_read(eeb_ctx* ctx, char* json_out, int64_t cap);
/* Per-CTA stamps (ns from the step's first start; -1 = none) of launch
 * `launch` of the last stamped step, CTAs [0, n) in linear block order. */
eeb_status eeb_debug_stamps_cta(eeb_ctx* ctx, int launch, int64_t* start_ns, int64_t* end_ns, int64_t* wait_ns,
                                int64_t* mark_ns,
                                int n);

/* Test/diagnostic hooks (not used on the serving path). */
eeb_status eeb_debug_last_logits(eeb_ctx* ctx, int head, float* host_out, int64_t n);  /* [batch][vocab] of one head, when retained */
eeb_status eeb_debug_retain_logits(eeb_ctx* ctx, int enable);
eeb_status eeb_debug_read_weight(eeb_ctx* ctx, int model, int tensor, int layer, int64_t offset,
                                 int64_t n, float* host_out);
eeb_status eeb_debug_read_kv(eeb_ctx* ctx, int model, int layer, int slot, int pos, float* host_k,
                             float* host_v);
/* K/V of positions [pos0, pos0 + n_pos) of one slot at one layer, as f32
 * [n_pos][n_kv_heads * head_dim] (either output may be null). */
eeb_status eeb_debug_read_kv_span(eeb_ctx* ctx, int model, int layer, int slot, int pos0, int n_pos,
                                  float* host_k, float* host_v);

/* Run one decode GEMM y[b][n] = sum_k x[b][k] * w[n][k] through a given tier
 * (1 CUDA cores, 2 tcgen05) with an epilogue mode (0 store f32, 1 residual add
 * onto zeros, 2 relu, 3 swiglu).  w, x are host arrays in the dtype (f32 or
 * bf16 bit patterns); y is host f32, [batch][n] (or [batch][n/2] for swiglu). */
eeb_status eeb_debug_gemm(eeb_ctx* ctx, int tier, int dtype, int n, int k, int batch, int mode,
                          const void* w_host, const void* x_host, float* y_host);

/* Steady-state timing of one decode GEMM shape: `iters` back-to-back launches
 * (PDL-chained, like inside a step) on device-resident random data; returns the
 * mean milliseconds per launch (CUDA events on the context stream). */
eeb_status eeb_debug_bench_gemm(eeb_ctx* ctx, int tier, int n, int k, int batch, int iters, double* ms_out);


/* Per-kernel timing of the last step (CUDA events on the context stream).
 * names: "gemm", "attention", "exit_head", ... ; returns total ms. */
eeb_status eeb_profile_enable(eeb_ctx* ctx, int enable);
eeb_status eeb_profile_read(eeb_ctx* ctx, char* json_out, int64_t cap);

/* Stream handle as an opaque pointer (cudaStream_t) for callers that want to
 * order their own work (e.g. torch) behind the step. */
void* eeb_stream(eeb_ctx* ctx);

/* NCCL histogram all-reduce across replicas at profiling boundaries
 * (SURVEY §8e): sums `n` int64 counters and one double in place.  The
 * communicator is created from a caller-distributed unique id. */
eeb_status eeb_nccl_unique_id(uint8_t* id128);
eeb_status eeb_nccl_init(eeb_ctx* ctx, const uint8_t* id128, int nranks, int rank);
eeb_status eeb_profile_allreduce(eeb_ctx* ctx, int64_t* counters, int n, double* sum_neg_logprob);

/* Peer-memory tensor parallelism (C5 over NVLink / NVSwitch, no NCCL on the
 * step's data path).  Each rank context of a tp_size > 1 model allocates one
 * exchange buffer (eeb_tp_px_alloc: returns its device pointer and a CUDA IPC
 * handle, 64 bytes), the caller distributes them (one process per GPU: the
 * IPC handles; ranks of one process: the pointers), and every rank attaches
 * the full set in rank order (eeb_tp_px_attach; peer_ptrs[p] may be null
 * where ipc_handles64 + 64 p is given; the own entry is ignored).  From then
 * on each row-parallel O / down GEMM is followed by ONE kernel that
 * reduce-scatters the partial planes across the ranks through peer memory,
 * all-gathers the reduced rows, and applies the residual add + RMSNorm
 * (tp_norm), and the vocab-parallel exit-head partials are all-gathered by a
 * peer-memory copy kernel.  Every rank must issue the same sequence of steps
 * and prefills (as with NCCL).  Replaces the reference's per-token model call
 * for a model served over several GPUs (engine.hpp:325-398). */
eeb_status eeb_tp_px_alloc(eeb_ctx* ctx, int model, void** dev_ptr, uint8_t* ipc_handle64);
eeb_status eeb_tp_px_attach(eeb_ctx* ctx, int model, int nranks, void* const* peer_ptrs,
                            const uint8_t* ipc_handles64);

#ifdef __cplusplus
}
#endif
#endif /* EEB_H_ */
