// eeserve/backend.hpp — where the decode step gets its exit-head verdicts.
//
// In the reference, Simulator::serve_one reads them from the trace
// (`tok.for_model(model)`, /root/reference/proj/include/eeserve/engine.hpp:345)
// and applies the token policy (:349-366).  Here that seam is an interface:
//   * CudaBackend  — the B200 decode step through the C ABI (include/eeb/eeb.h);
//   * TraceBackend — replays reference-format ModelTokenRecords (exactly the
//                    reference's semantics; used to cross-check the engine).
// Both return, per row, the observation the policy picked plus the
// breached / unchanged flags, and the step's exit histogram.
#pragma once

#include <chrono>
#include <functional>
#include <set>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "eeb/eeb.h"
#include "eeserve/model_spec.hpp"
#include "eeserve/trace.hpp"

namespace eeserve {

/// ↔ Simulator::TokenPolicy (engine.hpp:156) + the all-heads profiling pass.
enum class TokenPolicy { flat = EEB_FLAT, introspective = EEB_INTROSPECTIVE, full_depth = EEB_FULL_DEPTH,
                         profile = EEB_PROFILE };

struct StepRows {
    std::vector<int32_t> slots, tokens, positions;
    std::vector<std::int64_t> request_ids;  // trace backend: which request...
    std::vector<int32_t> token_index;       // ...and which of its tokens
    int size() const { return (int)slots.size(); }
};

struct StepOutcome {
    std::vector<ExitObservation> obs;      // per row: the observation the policy used
    std::vector<int> exit_layer;           // per row (flat: the serving depth)
    std::vector<uint8_t> breached, unchanged;  // unchanged: 1/0, 2 = unknown
    std::vector<std::int64_t> hist;        // per exit head
    std::int64_t n_breached = 0;
    double sum_logprob = 0.0;
    std::vector<ModelTokenRecord> records;  // profile policy: every head per row
    double seconds = 0.0;                   // measured step wall time
};

/// Prompts of a batch: sequence k = `prompts[k]` into KV slot `slots[k]`.
struct PrefillRows {
    std::vector<int32_t> slots;
    std::vector<std::vector<int32_t>> prompts;
    int size() const { return (int)slots.size(); }
};

/// A finished load: measured seconds and bytes moved (0 = not measured; the
/// engine then charges the reference's modelled bytes / bandwidth).
struct LoadResult {
    double seconds = 0.0;
    std::int64_t bytes = 0;
};

class DecodeBackend {
public:
    virtual ~DecodeBackend() = default;
    virtual void register_model(const ModelSpec& spec, int max_slots, int max_seq_len) = 0;
    /// Greedy loader ↔ do_load (engine.hpp:197-216): make layers [1, depth] resident.
    virtual LoadResult load(const std::string& model, int depth) = 0;
    /// Prefill ↔ serve_one's prefill phase (engine.hpp:333-341): the prompts'
    /// KV through layers 1..depth.  Returns the measured seconds (0 = modelled).
    virtual double prefill(const std::string& model, int depth, const PrefillRows& rows) = 0;
    virtual StepOutcome step(const std::string& model, int depth, TokenPolicy policy, double th,
                             const StepRows& rows) = 0;
    /// Continuous batching: the request in `slot` finished; its KV (pages) may
    /// be reused by the next request admitted into the slot.
    virtual void release(const std::string& model, int slot) { (void)model, (void)slot; }
};

// ---------------------------------------------------------------------------
// CUDA backend (C ABI).
// ---------------------------------------------------------------------------
class CudaBackend final : public DecodeBackend {
public:
    /// host_tier: keep every registered model's layers in pinned host memory
    /// and load by asynchronous H2D copies from it (the HELIOS loader);
    /// otherwise layers are materialised on device from the seed.
    explicit CudaBackend(int device = 0, bool host_tier = false) : host_tier_(host_tier) {
        throw_if_error(eeb_create(device, &ctx_), "eeb_create");
    }
    /// Paged KV pool for models registered after this call (eeb_kv_configure_pages):
    /// n_pages pages of page_size positions instead of max_slots x max_seq_len
    /// (bf16 models with head_dim 64 or 128; other models keep the slot pool).
    /// n_pages = 0: enough pages for every slot the engine sized from the
    /// memory model (max_slots x ceil(max_seq_len / page_size)).
    void set_kv_pages(int page_size, int n_pages = 0) {
        kv_page_ = page_size;
        kv_pages_ = n_pages;
    }
    ~CudaBackend() override { eeb_destroy(ctx_); }
    CudaBackend(const CudaBackend&) = delete;
    CudaBackend& operator=(const CudaBackend&) = delete;

    void register_model(const ModelSpec& spec, int max_slots, int max_seq_len) override {
        const Architecture& a = spec.arch;
        eeb_model_desc d{};
        d.num_layers = spec.num_layers;
        d.d_model = a.d_model;
        d.n_heads = a.n_heads;
        d.n_kv_heads = a.n_kv_heads;
        d.d_ffn = a.d_ffn;
        d.vocab = a.vocab;
        d.n_exits = (int32_t)spec.exit_layers.size();
        std::vector<int32_t> exits(spec.exit_layers.begin(), spec.exit_layers.end());
        d.exit_layers = exits.data();
        d.exit_coverage = a.exit_coverage.empty() ? nullptr : a.exit_coverage.data();
        d.design_th = a.design_th;
        d.dtype = a.dtype;
        d.mlp_kind = a.mlp_kind;
        d.max_slots = max_slots;
        d.max_seq_len = max_seq_len;
        d.seed = a.seed;
        int h = -1;
        throw_if_error(eeb_model_register(ctx_, &d, &h), "eeb_model_register");
        handles_[spec.id] = {h, spec};
        // the paged pool serves bf16 models with head_dim 64 / 80 / 128 (the
        // decode and prefill attention kernels walk page tables); others keep
        // the slot pool
        const int hd = a.n_heads > 0 ? a.d_model / a.n_heads : 0;
        if (kv_page_ > 0 && a.dtype == EEB_BF16 && (hd == 64 || hd == 80 || hd == 128))
            throw_if_error(eeb_kv_configure_pages(ctx_, h, kv_page_,
                                                  kv_pages_ > 0 ? kv_pages_
                                                                : max_slots * ((max_seq_len + kv_page_ - 1) / kv_page_)),
                           "eeb_kv_configure_pages");
        if (host_tier_) {
            throw_if_error(eeb_host_stage(ctx_, h, spec.num_layers), "eeb_host_stage");
            // device blocks for every depth the engine may load, allocated now (setup)
            throw_if_error(eeb_weight_reserve(ctx_, h, spec.num_layers), "eeb_weight_reserve");
        }
    }

    void release(const std::string& model, int slot) override {
        throw_if_error(eeb_kv_release(ctx_, handle(model).h, slot), "eeb_kv_release");
    }

    LoadResult load(const std::string& model, int depth) override {
        const int h = handle(model).h;
        LoadResult r;
        if (!host_tier_) {
            const auto t0 = std::chrono::steady_clock::now();
            throw_if_error(eeb_load_layers(ctx_, h, depth), "eeb_load_layers");
            r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return r;
        }
        int before = 0;
        throw_if_error(eeb_loaded_depth(ctx_, h, &before), "eeb_loaded_depth");
        throw_if_error(eeb_load_layers_async(ctx_, h, depth), "eeb_load_layers_async");
        if (depth > before) throw_if_error(eeb_load_wait(ctx_, h, &r.seconds, &r.bytes), "eeb_load_wait");
        return r;
    }

    double prefill(const std::string& model, int depth, const PrefillRows& rows) override {
        std::vector<int32_t> start(rows.size(), 0), lens, toks;
        for (const auto& p : rows.prompts) {
            lens.push_back((int32_t)p.size());
            toks.insert(toks.end(), p.begin(), p.end());
        }
        if (toks.empty()) return 0.0;
        const auto t0 = std::chrono::steady_clock::now();
        throw_if_error(eeb_prefill(ctx_, handle(model).h, depth, rows.size(), rows.slots.data(), start.data(),
                                   lens.data(), toks.data()),
                       "eeb_prefill");
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }

    StepOutcome step(const std::string& model, int depth, TokenPolicy policy, double th,
                     const StepRows& rows) override {
        const Entry& e = handle(model);
        const int b = rows.size(), ne = (int)e.spec.exit_layers.size();
        StepOutcome out;
        std::vector<int32_t> exit_layer(b), tok(b);
        std::vector<float> conf(b), logp(b);
        out.breached.resize(b);
        out.unchanged.resize(b);
        out.hist.resize(ne);
        std::vector<int32_t> htok;
        std::vector<float> hconf, hlogp;
        eeb_step_out o{};
        o.exit_layer = exit_layer.data();
        o.token_id = tok.data();
        o.confidence = conf.data();
        o.logprob = logp.data();
        o.breached = out.breached.data();
        o.unchanged = out.unchanged.data();
        o.hist = out.hist.data();
        o.n_breached = &out.n_breached;
        o.sum_logprob = &out.sum_logprob;
        if (policy == TokenPolicy::profile) {
            htok.resize((size_t)b * ne);
            hconf.resize((size_t)b * ne);
            hlogp.resize((size_t)b * ne);
            o.head_token = htok.data();
            o.head_confidence = hconf.data();
            o.head_logprob = hlogp.data();
        }
        const auto t0 = std::chrono::steady_clock::now();
        throw_if_error(eeb_decode_step(ctx_, e.h, depth, (int)policy, (float)th, b, rows.slots.data(),
                                       rows.tokens.data(), rows.positions.data(), &o),
                       "eeb_decode_step");
        out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out.exit_layer.assign(exit_layer.begin(), exit_layer.end());
        out.obs.resize(b);
        for (int i = 0; i < b; ++i) {
            // The head the policy used: its layer is the exit layer except in
            // flat mode between heads (observation_for_depth's fallback).
            int layer = exit_layer[i];
            if (policy == TokenPolicy::flat) layer = observation_layer_for_depth(e.spec, depth);
            out.obs[i] = ExitObservation{layer, tok[i], (double)conf[i], (double)logp[i]};
        }
        if (policy == TokenPolicy::profile) {
            out.records.resize(b);
            for (int i = 0; i < b; ++i) {
                ModelTokenRecord& r = out.records[i];
                for (int k = 0; k < ne; ++k)
                    r.observations.push_back({e.spec.exit_layers[k], htok[(size_t)i * ne + k],
                                              (double)hconf[(size_t)i * ne + k], (double)hlogp[(size_t)i * ne + k]});
                r.final_token_id = r.observations.back().token_id;
            }
        }
        return out;
    }

    eeb_ctx* context() const { return ctx_; }

private:
    int kv_page_ = 0, kv_pages_ = 0;
    struct Entry {
        int h;
        ModelSpec spec;
    };
    const Entry& handle(const std::string& id) const {
        const auto it = handles_.find(id);
        if (it == handles_.end()) throw DomainError("model '" + id + "' is not registered with the backend");
        return it->second;
    }
    static int observation_layer_for_depth(const ModelSpec& spec, int depth) {
        int best = -1;
        for (int l : spec.exit_layers)
            if (l <= depth) best = l;
        if (best < 0) throw DomainError("no observation at or below layer " + std::to_string(depth));
        return best;
    }
    eeb_ctx* ctx_ = nullptr;
    bool host_tier_ = false;
    std::map<std::string, Entry> handles_;
};

// The reference's per-token rule (engine.hpp:349-366) applied to one row's
// record: the observation the policy uses, the exit layer, the breach and
// unchanged flags, appended to `out`.
inline void apply_token_policy(const ModelSpec& spec, const ModelTokenRecord& rec, int depth, TokenPolicy policy,
                               double th, StepOutcome& out) {
    const ExitObservation* obs = nullptr;
    int exit_layer = 0;
    bool breached = false;
    switch (policy) {
        case TokenPolicy::flat:
            obs = &observation_for_depth(rec, depth);
            exit_layer = depth;
            breached = obs->confidence < th;
            break;
        case TokenPolicy::full_depth:
            obs = &rec.observations.back();
            exit_layer = spec.num_layers;
            break;
        default:
            obs = &earliest_confident_obs(rec, th);
            exit_layer = obs->layer;
            breached = obs->confidence < th;
            break;
    }
    if (out.hist.empty()) out.hist.assign(spec.exit_layers.size(), 0);
    out.obs.push_back(*obs);
    out.exit_layer.push_back(exit_layer);
    out.breached.push_back(breached ? 1 : 0);
    out.unchanged.push_back(obs->token_id == rec.final_token_id ? 1 : 0);
    out.hist[exit_index(spec.exit_layers, obs->layer)] += 1;
    out.n_breached += breached ? 1 : 0;
    out.sum_logprob += obs->logprob;
    if (policy == TokenPolicy::profile) out.records.push_back(rec);
}

// ---------------------------------------------------------------------------
// Profile backend: the reference's serve_one semantics over live GPU decode.
// Every step runs every exit head on the GPU at full depth (EEB_PROFILE: the
// ModelTokenRecord the reference would look up in its trace,
// engine.hpp:345) and applies the reference's token rule on the host, so a
// BatchedEngine over it reproduces Simulator::run on the records the GPU
// produces — the same decisions, exit tables and breach actions.  Times are
// the reference's modelled ones (loads bytes / bandwidth, prefill and decode
// per layer), so whole reports compare exactly.  Also a trace recorder: the
// records of every step can be collected and written as a reference trace.
// ---------------------------------------------------------------------------
class ProfileBackend final : public DecodeBackend {
public:
    explicit ProfileBackend(CudaBackend& gpu) : gpu_(gpu) {}
    void register_model(const ModelSpec& spec, int max_slots, int max_seq_len) override {
        specs_[spec.id] = spec;
        gpu_.register_model(spec, max_slots, max_seq_len);
    }
    LoadResult load(const std::string& model, int depth) override {
        // every head needs every layer: resident at full depth on first use
        if (depth > 0 && !full_.count(model)) {
            gpu_.load(model, specs_.at(model).num_layers);
            full_.insert(model);
        }
        return {};
    }
    double prefill(const std::string& model, int, const PrefillRows& rows) override {
        gpu_.prefill(model, specs_.at(model).num_layers, rows);  // full-depth KV (profiled decode attends it)
        return 0.0;
    }
    StepOutcome step(const std::string& model, int depth, TokenPolicy policy, double th,
                     const StepRows& rows) override {
        const ModelSpec& spec = specs_.at(model);
        const StepOutcome gpu = gpu_.step(model, 0, TokenPolicy::profile, th, rows);
        StepOutcome out;
        for (int i = 0; i < rows.size(); ++i) {
            apply_token_policy(spec, gpu.records[i], depth, policy, th, out);
            if (recorder) recorder(model, rows.request_ids[i], rows.token_index[i], gpu.records[i]);
        }
        return out;
    }
    void release(const std::string& model, int slot) override { gpu_.release(model, slot); }

    /// Called with every row's record (model, request id, token index, record).
    std::function<void(const std::string&, std::int64_t, int, const ModelTokenRecord&)> recorder;

private:
    CudaBackend& gpu_;
    std::map<std::string, ModelSpec> specs_;
    std::set<std::string> full_;
};

// ---------------------------------------------------------------------------
// Trace backend: the reference's token oracle, batched.
// ---------------------------------------------------------------------------
class TraceBackend final : public DecodeBackend {
public:
    explicit TraceBackend(const Trace& trace) {
        for (const auto& r : trace.requests) by_id_[r.request_id] = &r;
    }
    void register_model(const ModelSpec& spec, int, int) override { specs_[spec.id] = spec; }
    LoadResult load(const std::string&, int) override { return {}; }
    double prefill(const std::string&, int, const PrefillRows&) override { return 0.0; }

    StepOutcome step(const std::string& model, int depth, TokenPolicy policy, double th,
                     const StepRows& rows) override {
        const ModelSpec& spec = specs_.at(model);
        StepOutcome out;
        out.hist.assign(spec.exit_layers.size(), 0);
        for (int i = 0; i < rows.size(); ++i) {
            const TraceRequest& req = *by_id_.at(rows.request_ids[i]);
            apply_token_policy(spec, req.tokens.at(rows.token_index[i]).for_model(model), depth, policy, th, out);
        }
        return out;
    }

private:
    std::map<std::int64_t, const TraceRequest*> by_id_;
    std::map<std::string, ModelSpec> specs_;
};

}  // namespace eeserve
