/*
 * eeb_oracle.h — CPU oracle for the batched early-exit decode step.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link or
 * call this; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * reference arm use it, as the checker.
 *
 * It restates, straight-line and in plain C:
 *   - the synthetic model definition (docs: DESIGN.md §3; product code:
 *     paper_2504_10724_b200/csrc/synth.cuh) — independently re-implemented;
 *   - the decoder: pre-RMSNorm blocks, RoPE attention over a KV cache, ReLU /
 *     SwiGLU MLP, with the same rounding points as the device path (activations
 *     fed to a matrix product and the KV cache are rounded to the model dtype;
 *     residual stream f32); dot products accumulate in f64;
 *   - the exit-head semantics of the reference (HELIOS simulator):
 *       confidence = max softmax prob, logprob = log p(argmax) — SPEC.md:106;
 *       earliest_confident_obs — /root/reference/proj/include/eeserve/trace.hpp:69-76;
 *       observation_for_depth  — trace.hpp:86-97;
 *       breached = conf < th, full depth never breaches — engine.hpp:349-365;
 *       unchanged = head token == final token — engine.hpp:366.
 * The reference itself computes no logits (it is a trace-driven simulator), so
 * the tensor arithmetic here has no reference to pin against: DESIGN.md says
 * "parity unpinned" for logits; the decision layer is pinned against the
 * reference's own KATs and against the compiled reference (oracle/_ref).
 */
#ifndef EEB_ORACLE_H_
#define EEB_ORACLE_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int num_layers, d_model, n_heads, n_kv_heads, d_ffn, vocab;
    int n_exits;
    int exit_layers[64];
    float exit_coverage[64];
    float design_th;
    int dtype;      /* 0 f32, 1 bf16 */
    int mlp_kind;   /* 0 relu, 1 swiglu */
    int max_slots, max_seq_len;
    uint64_t seed;
    float rope_theta, norm_eps;
} orc_desc;

typedef struct orc_model orc_model;

orc_model* orc_create(const orc_desc* d, int threads);
void orc_destroy(orc_model* m);
/* materialise weights for layers [1, depth] (base weights always) */
int orc_load(orc_model* m, int depth);
float orc_alpha(const orc_model* m, int e);
/* One element of a tensor (kinds as in the product: layer 0..5, base 100 emb,
 * 200+e head, 300+e head norm), already rounded to the model dtype. */
float orc_weight(const orc_model* m, int tensor, int layer, int64_t index);

/* Outputs per caller row (arrays of batch), profile arrays [batch][n_exits].
 * logits_out (optional): [n_exits][batch][vocab], filled for every head
 * evaluated on a row (rows not evaluated at a head are left untouched). */
typedef struct {
    int32_t* exit_layer;
    int32_t* token_id;
    float* confidence;
    float* logprob;
    uint8_t* breached;
    uint8_t* unchanged;
    int64_t* hist;
    int64_t* n_breached;
    double* sum_logprob;
    int32_t* head_token;
    float* head_confidence;
    float* head_logprob;
    float* logits_out;
} orc_out;

int orc_decode_step(orc_model* m, int serving_depth, int policy, float th, int batch,
                    const int32_t* slots, const int32_t* tokens, const int32_t* positions,
                    orc_out* out);
/* The reference's per-token exit rule over one complete ModelTokenRecord
 * (policy 0 flat / 1 introspective / 2 full depth / 3 = 1), see eeb_oracle.c. */
typedef struct { int index, exit_layer, breached, unchanged; } orc_decision;
int orc_decide(int policy, int n, const int32_t* layers, const int32_t* toks, const float* confs, float th,
               int depth, int num_layers, orc_decision* out);
/* K/V of one position, [n_kv_heads][head_dim] each. */
int orc_read_kv(const orc_model* m, int layer, int slot, int pos, float* k, float* v);
/* Whole tensors (kinds as orc_weight): get returns the element count (copies
 * min(n, count) when out is set); set replaces all of it (rounded to the dtype). */
int64_t orc_tensor_get(orc_model* m, int tensor, int layer, float* out, int64_t n);
int orc_tensor_set(orc_model* m, int tensor, int layer, const float* src, int64_t n);
/* Import K/V of positions [pos0, pos0+n) ([n][n_kv_heads*head_dim] each) at one layer. */
int orc_write_kv(orc_model* m, int layer, int slot, int pos0, int n, const float* k, const float* v);
/* Synthetic full-depth KV for positions [0, n) of a slot (CPU-baseline context). */
int orc_fill_kv_synthetic(orc_model* m, int slot, int n, uint64_t seed);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
