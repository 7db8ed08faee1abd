// eeserve/engine.hpp — the batched serving loop around the decode step.
//
// The reference's Simulator (/root/reference/proj/include/eeserve/engine.hpp:108-399)
// serves requests one at a time (batch 1, :104-107) and reads every token's
// exit verdicts from a trace.  BatchedEngine keeps its control flow — mode
// dispatch (:139-151), evaluation cycles that profile every candidate at full
// depth with the introspective rule (:243-278), replanning (:280-299), breach
// actions queued by decide_action and applied at the next request boundary
// (:301-323, :381-385) — but advances up to `max_batch` requests per decode
// step through a DecodeBackend (every in-flight request
// moves one token per step).  Metrics follow metrics.hpp:85-93: the tokens of
// one step share one timestamp, so a step's wall time is charged once.
//
// With max_batch = 1 and the TraceBackend the engine reproduces the
// reference's exit tables and breach/switch decisions (tests/cpp).
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "eeserve/backend.hpp"
#include "eeserve/events.hpp"
#include "eeserve/memory_model.hpp"
#include "eeserve/pht.hpp"
#include "eeserve/policy.hpp"

namespace eeserve {

enum class Mode { vanilla, ee_single, helios };

struct ModeSpec {
    Mode kind = Mode::helios;
    std::string model;  // pinned modes
};

struct RequestSpec {
    std::int64_t request_id = 0;
    int prompt_len = 0;
    int num_tokens = 0;
};

struct EngineConfig {
    MemoryConfig mem;
    PolicyConfig policy;
    ModeSpec mode;
    int max_batch = 64;
    int max_seq_len = 256;
    std::uint64_t token_seed = 20260819;
    bool prefill = true;  // run the prompt through the backend (real KV); off for trace replay
    bool record_events = false;  // keep the reference-format event log (events.hpp) in the report
    // Continuous batching: a finished request's slot is
    // released (DecodeBackend::release) and the next queued request is
    // prefilled into it while the others keep decoding; admission stops at a
    // policy boundary (reassessment due or a pending breach action) and the
    // in-flight requests drain first, so actions still apply at request
    // boundaries (engine.hpp:143).  max_batch = 1 is the reference's loop.
    bool continuous = false;
    // Teacher-forced input-token law (prompt and decode inputs); unset =
    // synthetic_token(token_seed, ...).  serve_c3's drift workload picks
    // tokens by their synthetic difficulty so breaches happen on the GPU.
    std::function<int32_t(std::int64_t request_id, int position, int vocab)> token_fn;
};

struct RequestTiming {  // ↔ the request's TTFT (engine.hpp:333-337) and its tokens' TPOT
    std::int64_t request_id = 0;
    double ttft_s = 0.0;
    double tpot_sum_s = 0.0;
    int tokens = 0;
};

struct EngineReport {
    std::int64_t tokens = 0;
    std::int64_t steps = 0;
    double decode_wall_s = 0.0;
    double throughput_tok_s = 0.0;
    double perplexity = 0.0;
    double unchanged_fraction = 0.0;  // over tokens whose final-head token is known
    std::map<std::string, std::map<int, std::int64_t>> exit_counts;
    std::map<std::string, std::map<int, double>> exit_table;  // percent of tokens
    int achieved_batch_size = 0;
    std::int64_t ld_count = 0, sw_count = 0, eval_cycles = 0;
    std::vector<std::pair<std::string, int>> serving_history;  // (model, depth) per served batch
    double load_s = 0.0;              // loader stalls (measured, or bytes / bandwidth when not measured)
    std::int64_t load_bytes = 0;
    double prefill_s = 0.0;
    std::vector<RequestTiming> requests;
    double mean_ttft_s = 0.0, mean_tpot_s = 0.0;
    std::vector<EngineEvent> events;  // EngineConfig::record_events
    Pht pht;
};

/// Teacher-forced synthetic token for (request, position): a splitmix64 hash,
/// the same request-keyed substream idea as the reference generator
/// (rng.hpp:9-38, generator.hpp:319-323).
inline int32_t synthetic_token(std::uint64_t seed, std::int64_t request_id, int position, int vocab) {
    std::uint64_t z = seed ^ (0x9e3779b97f4a7c15ULL * (std::uint64_t)(request_id + 1)) ^
                      (0xd1b54a32d192ed03ULL * (std::uint64_t)(position + 7));
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return (int32_t)(z % (std::uint64_t)vocab);
}

class BatchedEngine {
public:
    BatchedEngine(const ModelRepository& repo, DecodeBackend& backend, EngineConfig cfg)
        : repo_(repo), be_(backend), cfg_(std::move(cfg)) {}

    /// Validate the configuration, pick the candidates and register them with
    /// the backend (device KV pool sized from the memory model; the host tier
    /// stages their layers).  run() calls it when the caller did not, so a
    /// caller may time setup and serving separately.
    void prepare() {
        if (prepared_) return;
        validate_memory_config(cfg_.mem);
        validate_policy_config(cfg_.policy);
        if (cfg_.max_batch < 1) throw ValidationError("engine: max_batch must be at least 1");
        const PolicyConfig& pol = cfg_.policy;
        if (cfg_.mode.kind == Mode::helios) {
            candidates_ = select_candidates(repo_, pol.slo, cfg_.mem, pol.k);
        } else {
            if (!repo_.has(cfg_.mode.model))
                throw ValidationError("mode model '" + cfg_.mode.model + "' is not in the repository");
            candidates_ = {cfg_.mode.model};
        }
        for (const auto& id : candidates_) {
            const int slots = slots_for(repo_.at(id));
            slots_[id] = slots;
            be_.register_model(repo_.at(id), slots, cfg_.max_seq_len);
        }
        prepared_ = true;
    }

    /// Decode slots (the device KV pool's rows) for a model: the memory
    /// model's batch capacity at full depth with only this model resident
    /// (max_batch_size over kv_budget_bytes, memory_model.hpp:53-72), capped
    /// by max_batch; at least 1 (load_for_eval raises CapacityError when not
    /// even one sequence fits, engine.hpp:231-233).
    int slots_for(const ModelSpec& spec) const {
        MemoryState alone;
        alone.loaded_depth[spec.id] = spec.num_layers;
        const int cap =
            max_batch_size(spec, spec.num_layers, kv_budget_bytes(cfg_.mem, alone, repo_), cfg_.mem.max_seq_len);
        return std::max(1, std::min(cfg_.max_batch, cap));
    }
    int slots(const std::string& id) const {
        auto it = slots_.find(id);
        return it == slots_.end() ? cfg_.max_batch : it->second;
    }

    EngineReport run(const std::vector<RequestSpec>& reqs) {
        prepare();
        const PolicyConfig& pol = cfg_.policy;
        if (reqs.empty()) return finish();
        if (cfg_.mode.kind == Mode::helios) {
            since_eval_ = pol.ri;  // evaluate before serving anything (engine.hpp:130)
        } else {
            serving_ = cfg_.mode.model;
            depth_ = repo_.at(serving_).num_layers;
            do_load(serving_, depth_, "startup");
        }
        const TokenPolicy tp = cfg_.mode.kind == Mode::vanilla    ? TokenPolicy::full_depth
                               : cfg_.mode.kind == Mode::ee_single ? TokenPolicy::introspective
                                                                   : TokenPolicy::flat;
        while (cursor_ < reqs.size()) {
            if (cfg_.mode.kind == Mode::helios && should_reassess(since_eval_, pol)) {
                eval_cycle(reqs);
                continue;
            }
            if (pending_) apply_pending();
            if (cfg_.continuous) {
                serve_continuous(reqs, serving_, depth_, tp);
                continue;
            }
            const size_t n = std::min<size_t>(slots(serving_), reqs.size() - cursor_);
            std::vector<const RequestSpec*> batch;
            for (size_t i = 0; i < n; ++i) batch.push_back(&reqs[cursor_ + i]);
            cursor_ += n;
            since_eval_ += (std::int64_t)n;
            serve_batch(batch, serving_, depth_, tp, false);
        }
        return finish();
    }

private:
    const ModelRepository& repo_;
    DecodeBackend& be_;
    EngineConfig cfg_;
    bool prepared_ = false;
    std::map<std::string, int> slots_;
    std::vector<std::string> candidates_;
    MemoryState mem_;
    std::string serving_;
    int depth_ = 0;
    Pht pht_;
    BreachTracker breach_;
    std::optional<ActionPlan> pending_;
    std::int64_t since_eval_ = 0;
    size_t cursor_ = 0;
    EngineReport rep_;
    double sum_logprob_ = 0.0;
    std::int64_t unchanged_ = 0, unchanged_known_ = 0;
    double pending_stall_s_ = 0.0;  // loads charged to the next batch's TTFT (engine.hpp:205-207, :336)
    double clock_ = 0.0;            // serving clock of the event log (s)

    int32_t token(std::int64_t request_id, int position, int vocab) const {
        return cfg_.token_fn ? cfg_.token_fn(request_id, position, vocab)
                             : synthetic_token(cfg_.token_seed, request_id, position, vocab);
    }

    void emit(const char* kind, const JsonFields& f) {
        if (cfg_.record_events) rep_.events.push_back({clock_, kind, f.body()});
    }

    void do_load(const std::string& id, int target, const std::string& reason) {
        const int from = mem_.depth_of(id);
        if (from == target) return;
        const std::int64_t modelled = load_delta_bytes(repo_.at(id), from, target);
        apply_load(mem_, repo_, cfg_.mem, id, target);  // CapacityError leaves state untouched
        const LoadResult lr = be_.load(id, target);
        // growth pays the transfer (measured when the backend moved real bytes);
        // shrink and eviction are free (engine.hpp:197-199)
        const double dur = target < from ? 0.0 : lr.seconds > 0.0 ? lr.seconds : load_seconds(modelled, cfg_.mem);
        rep_.load_s += dur;
        const std::int64_t moved = lr.bytes > 0 ? lr.bytes : std::max<std::int64_t>(0, modelled);
        rep_.load_bytes += moved;
        pending_stall_s_ += dur;
        clock_ += dur;
        emit("weights_load", JsonFields()
                                 .str("model", id)
                                 .i64("from_depth", from)
                                 .i64("to_depth", target)
                                 .i64("bytes", moved)
                                 .num("duration_s", dur)
                                 .str("reason", reason)
                                 .i64("loaded_bytes_after", weights_loaded_bytes(mem_, repo_))
                                 .num("energy_mwh", 0.0));
        if (reason == "breach_load_more") ++rep_.ld_count;
    }

    void load_for_eval(const std::string& id) {  // engine.hpp:220-234
        const ModelSpec& spec = repo_.at(id);
        MemoryState trial = mem_;
        trial.loaded_depth[id] = spec.num_layers;
        if (weights_loaded_bytes(trial, repo_) > cfg_.mem.capacity_bytes - cfg_.mem.reserve_bytes) {
            std::vector<std::string> others;
            for (const auto& [o, d] : mem_.loaded_depth)
                if (o != id && d > 0) others.push_back(o);
            for (const auto& o : others) do_load(o, 0, "evict");
        }
        do_load(id, spec.num_layers, "eval");
        if (max_batch_size(spec, spec.num_layers, kv_budget_bytes(cfg_.mem, mem_, repo_), cfg_.mem.max_seq_len) < 1)
            throw CapacityError("cannot fit one sequence while profiling '" + id + "'");
    }

    void eval_cycle(const std::vector<RequestSpec>& reqs) {  // engine.hpp:243-278
        ++rep_.eval_cycles;
        pending_.reset();
        breach_.reset();
        since_eval_ = 0;
        emit("reassess_start", JsonFields().i64("cycle", rep_.eval_cycles));
        for (const std::string& id : candidates_) {
            if (cursor_ >= reqs.size()) break;
            emit("eval_phase_start", JsonFields().str("model", id));
            pht_.reset(id);
            load_for_eval(id);
            const ModelSpec& spec = repo_.at(id);
            int served = 0;
            while (served < cfg_.policy.n_eval_requests && cursor_ < reqs.size()) {
                const size_t n = std::min<size_t>({(size_t)slots(id), reqs.size() - cursor_,
                                                   (size_t)(cfg_.policy.n_eval_requests - served)});
                std::vector<const RequestSpec*> batch;
                for (size_t i = 0; i < n; ++i) batch.push_back(&reqs[cursor_ + i]);
                cursor_ += n;
                served += (int)n;
                since_eval_ += (std::int64_t)n;  // evaluation requests count toward ri (serve_one, engine.hpp:331)
                serve_batch(batch, id, spec.num_layers, TokenPolicy::profile, true);
            }
            emit("eval_phase_end", JsonFields().str("model", id));
        }
        std::vector<std::string> profiled;
        for (const auto& id : candidates_)
            if (pht_.has(id)) profiled.push_back(id);
        if (profiled.empty()) {
            emit("reassess_end", JsonFields().i64("cycle", rep_.eval_cycles));
            return;
        }
        const ReplanResult plan = replan_after_eval(repo_, pht_, profiled, cfg_.policy, cfg_.mem);
        std::vector<std::string> drop;
        for (const auto& [id, d] : mem_.loaded_depth) {
            if (d <= 0) continue;
            bool keep = false;
            for (const auto& r : plan.residency) keep |= r.first == id;
            if (!keep) drop.push_back(id);
        }
        for (const auto& id : drop) do_load(id, 0, "reassess");
        for (const auto& [id, depth] : plan.residency) do_load(id, depth, "reassess");
        if (!serving_.empty() && serving_ != plan.serving_model)
            emit("model_switch", JsonFields().str("from", serving_).str("to", plan.serving_model).str("reason", "reassess"));
        serving_ = plan.serving_model;
        depth_ = plan.serving_depth;
        emit("reassess_end", JsonFields().i64("cycle", rep_.eval_cycles));
    }

    void apply_pending() {  // engine.hpp:301-323
        const ActionPlan plan = *pending_;
        pending_.reset();
        if (plan.kind != ActionKind::stay) {
            for (const auto& id : plan.evict) do_load(id, 0, "breach_evict");
            if (plan.kind == ActionKind::load_more) {
                do_load(plan.model_id, plan.serving_depth, "breach_load_more");
            } else {
                if (mem_.depth_of(plan.model_id) < plan.serving_depth)
                    do_load(plan.model_id, plan.serving_depth, "breach_switch");
                ++rep_.sw_count;
                emit("model_switch",
                     JsonFields().str("from", serving_).str("to", plan.model_id).str("reason", "breach_action"));
                serving_ = plan.model_id;
            }
            depth_ = plan.serving_depth;
        }
        breach_.reset();
    }

    std::vector<std::string> profiled_candidates() const {
        std::vector<std::string> out;
        for (const auto& id : candidates_)
            if (id == serving_ || pht_.has(id)) out.push_back(id);
        return out;
    }

    void serve_batch(const std::vector<const RequestSpec*>& batch, const std::string& model, int depth,
                     TokenPolicy tp, bool profile) {
        const ModelSpec& spec = repo_.at(model);
        const int vocab = spec.arch.vocab > 0 ? spec.arch.vocab : 1;
        rep_.serving_history.emplace_back(model, depth);
        const int b = (int)batch.size();
        int max_prompt = 0, max_tokens = 0;
        for (const auto* r : batch) {
            max_prompt = std::max(max_prompt, r->prompt_len);
            max_tokens = std::max(max_tokens, r->num_tokens);
        }
        // Prefill (engine.hpp:333-341): the prompts' KV through the layers the
        // step will run (the serving depth in flat mode, all layers otherwise).
        // TTFT = the pending loader stall + the prefill (engine.hpp:336).
        for (int i = 0; i < b; ++i) emit("request_start", JsonFields().i64("request_id", batch[i]->request_id));
        double prefill_s = 0.0;
        if (cfg_.prefill) {
            PrefillRows pr;
            for (int i = 0; i < b; ++i) {
                pr.slots.push_back(i);
                std::vector<int32_t> p(batch[i]->prompt_len);
                for (int k = 0; k < batch[i]->prompt_len; ++k)
                    p[k] = token(batch[i]->request_id, k, vocab);
                pr.prompts.push_back(std::move(p));
            }
            prefill_s = be_.prefill(model, tp == TokenPolicy::flat ? depth : spec.num_layers, pr);
        }
        if (prefill_s <= 0.0)  // modelled (engine.hpp:333-334): prompt_len x depth x t_prefill
            prefill_s = (double)max_prompt * depth * spec.t_prefill_per_layer_per_token_s;
        rep_.prefill_s += prefill_s;
        clock_ += prefill_s;
        for (int i = 0; i < b; ++i)
            emit("prefill", JsonFields()
                                .i64("request_id", batch[i]->request_id)
                                .str("model", model)
                                .i64("depth", depth)
                                .num("duration_s", prefill_s));
        const double ttft = pending_stall_s_ + prefill_s;
        pending_stall_s_ = 0.0;
        const size_t first_timing = rep_.requests.size();
        for (int i = 0; i < b; ++i) rep_.requests.push_back({batch[i]->request_id, ttft, 0.0, 0});
        // Decode: one token per in-flight request per step.
        for (int t = 0; t < max_tokens; ++t) {
            StepRows rows;
            for (int i = 0; i < b; ++i) {
                if (t >= batch[i]->num_tokens) continue;
                const int pos = batch[i]->prompt_len + t;
                rows.slots.push_back(i);
                rows.tokens.push_back(token(batch[i]->request_id, pos, vocab));
                rows.positions.push_back(pos);
                rows.request_ids.push_back(batch[i]->request_id);
                rows.token_index.push_back(t);
            }
            const StepOutcome o = be_.step(model, depth, tp, cfg_.policy.th, rows);
            double dur = o.seconds;
            if (dur <= 0.0) {  // modelled (trace backend): the step lasts as long as its deepest row
                int deepest = 0;
                for (int x : o.exit_layer) deepest = std::max(deepest, x);
                dur = deepest * spec.t_decode_per_layer_s;
            }
            clock_ += dur;  // every row of the step is emitted at the step's end (one t_s)
            for (int i = 0; cfg_.record_events && i < rows.size(); ++i)  // (no JSON built unless recorded)
                emit("token_emitted", JsonFields()
                                          .i64("request_id", rows.request_ids[i])
                                          .str("model", model)
                                          .i64("exit_layer", o.exit_layer[i])
                                          .boolean("breached", o.breached[i] != 0)
                                          .boolean("unchanged", o.unchanged[i] == 1)
                                          .num("duration_s", dur)
                                          .num("logprob", o.obs[i].logprob)
                                          .num("energy_mwh", o.exit_layer[i] * spec.energy_per_layer_per_token_mwh));
            consume(model, spec, tp, profile, rows, o, dur);
            for (int i = 0; i < b; ++i)
                if (t < batch[i]->num_tokens) {
                    rep_.requests[first_timing + i].tpot_sum_s += dur;
                    rep_.requests[first_timing + i].tokens += 1;
                }
        }
        for (int i = 0; i < b; ++i) {  // engine.hpp:387-395
            const RequestTiming& rt = rep_.requests[first_timing + i];
            const double tpot_mean = rt.tokens ? rt.tpot_sum_s / rt.tokens : 0.0;
            emit("request_complete", JsonFields()
                                         .i64("request_id", rt.request_id)
                                         .num("ttft_s", rt.ttft_s)
                                         .num("tpot_mean_s", tpot_mean)
                                         .num("latency_s", rt.ttft_s + tpot_mean * (double)rt.tokens)
                                         .i64("tokens", rt.tokens));
        }
    }

    // Continuous batching over the request queue from cursor_ (see EngineConfig::continuous).
    void serve_continuous(const std::vector<RequestSpec>& reqs, const std::string& model, int depth, TokenPolicy tp) {
        const ModelSpec& spec = repo_.at(model);
        const int vocab = spec.arch.vocab > 0 ? spec.arch.vocab : 1;
        rep_.serving_history.emplace_back(model, depth);
        struct Active {
            const RequestSpec* r;
            int slot;
            int t;          // tokens emitted so far
            size_t timing;  // index in rep_.requests
        };
        std::vector<Active> act;
        std::vector<int> free_slots;
        for (int s = slots(model) - 1; s >= 0; --s) free_slots.push_back(s);  // lowest slot first
        auto admissible = [&] {
            return cursor_ < reqs.size() && !pending_ &&
                   !(cfg_.mode.kind == Mode::helios && should_reassess(since_eval_, cfg_.policy));
        };
        auto complete = [&](const Active& a) {  // engine.hpp:387-395
            const RequestTiming& rt = rep_.requests[a.timing];
            const double tpot_mean = rt.tokens ? rt.tpot_sum_s / rt.tokens : 0.0;
            emit("request_complete", JsonFields()
                                         .i64("request_id", rt.request_id)
                                         .num("ttft_s", rt.ttft_s)
                                         .num("tpot_mean_s", tpot_mean)
                                         .num("latency_s", rt.ttft_s + tpot_mean * (double)rt.tokens)
                                         .i64("tokens", rt.tokens));
            be_.release(model, a.slot);
            free_slots.push_back(a.slot);
        };
        auto admit = [&] {
            std::vector<Active> fresh;
            while (!free_slots.empty() && admissible()) {
                fresh.push_back({&reqs[cursor_], free_slots.back(), 0, 0});
                free_slots.pop_back();
                ++cursor_;
                ++since_eval_;
            }
            if (fresh.empty()) return;
            for (const auto& a : fresh) emit("request_start", JsonFields().i64("request_id", a.r->request_id));
            double prefill_s = 0.0;
            int max_prompt = 0;
            for (const auto& a : fresh) max_prompt = std::max(max_prompt, a.r->prompt_len);
            if (cfg_.prefill) {
                PrefillRows pr;
                for (const auto& a : fresh) {
                    pr.slots.push_back(a.slot);
                    std::vector<int32_t> p(a.r->prompt_len);
                    for (int k = 0; k < a.r->prompt_len; ++k)
                        p[k] = token(a.r->request_id, k, vocab);
                    pr.prompts.push_back(std::move(p));
                }
                prefill_s = be_.prefill(model, tp == TokenPolicy::flat ? depth : spec.num_layers, pr);
            }
            if (prefill_s <= 0.0) prefill_s = (double)max_prompt * depth * spec.t_prefill_per_layer_per_token_s;
            rep_.prefill_s += prefill_s;
            clock_ += prefill_s;
            for (const auto& a : fresh)
                emit("prefill", JsonFields()
                                    .i64("request_id", a.r->request_id)
                                    .str("model", model)
                                    .i64("depth", depth)
                                    .num("duration_s", prefill_s));
            const double ttft = pending_stall_s_ + prefill_s;
            pending_stall_s_ = 0.0;
            for (auto& a : fresh) {
                a.timing = rep_.requests.size();
                rep_.requests.push_back({a.r->request_id, ttft, 0.0, 0});
                if (a.r->num_tokens <= 0) complete(a);
                else act.push_back(a);
            }
        };
        admit();
        while (!act.empty()) {
            // rows in ascending slot order (breach observation order, SURVEY §7 hard part 4)
            std::sort(act.begin(), act.end(), [](const Active& x, const Active& y) { return x.slot < y.slot; });
            StepRows rows;
            for (const auto& a : act) {
                const int pos = a.r->prompt_len + a.t;
                rows.slots.push_back(a.slot);
                rows.tokens.push_back(token(a.r->request_id, pos, vocab));
                rows.positions.push_back(pos);
                rows.request_ids.push_back(a.r->request_id);
                rows.token_index.push_back(a.t);
            }
            const StepOutcome o = be_.step(model, depth, tp, cfg_.policy.th, rows);
            double dur = o.seconds;
            if (dur <= 0.0) {
                int deepest = 0;
                for (int x : o.exit_layer) deepest = std::max(deepest, x);
                dur = deepest * spec.t_decode_per_layer_s;
            }
            clock_ += dur;
            for (int i = 0; cfg_.record_events && i < rows.size(); ++i)  // (no JSON built unless recorded)
                emit("token_emitted", JsonFields()
                                          .i64("request_id", rows.request_ids[i])
                                          .str("model", model)
                                          .i64("exit_layer", o.exit_layer[i])
                                          .boolean("breached", o.breached[i] != 0)
                                          .boolean("unchanged", o.unchanged[i] == 1)
                                          .num("duration_s", dur)
                                          .num("logprob", o.obs[i].logprob)
                                          .num("energy_mwh", o.exit_layer[i] * spec.energy_per_layer_per_token_mwh));
            consume(model, spec, tp, false, rows, o, dur);
            std::vector<Active> still;
            for (auto& a : act) {
                RequestTiming& rt = rep_.requests[a.timing];
                rt.tpot_sum_s += dur;
                rt.tokens += 1;
                if (++a.t >= a.r->num_tokens) complete(a);
                else still.push_back(a);
            }
            act.swap(still);
            admit();
        }
    }

    void consume(const std::string& model, const ModelSpec& spec, TokenPolicy tp, bool profile,
                 const StepRows& rows, const StepOutcome& o, double dur) {
        const int n = rows.size();
        rep_.tokens += n;
        rep_.steps += 1;
        rep_.decode_wall_s += dur;
        rep_.achieved_batch_size = std::max(rep_.achieved_batch_size, n);
        for (int i = 0; i < n; ++i) {
            rep_.exit_counts[model][o.exit_layer[i]] += 1;
            sum_logprob_ += o.obs[i].logprob;
            if (o.unchanged[i] != 2) {
                ++unchanged_known_;
                unchanged_ += o.unchanged[i];
            }
        }
        if (profile) {  // record_token per row == record_step over the step histogram
            std::vector<std::int64_t> hist(spec.exit_layers.size(), 0);
            double sl = 0.0;
            for (int i = 0; i < n; ++i) {
                hist[exit_index(spec.exit_layers, o.exit_layer[i])] += 1;
                sl += o.obs[i].logprob;
            }
            record_step(pht_, spec, hist, sl, dur);
        }
        if (tp == TokenPolicy::flat && cfg_.mode.kind == Mode::helios) {
            for (int i = 0; i < n; ++i)  // ascending slot order (SURVEY §7 hard part 4)
                if (observe_token(breach_, o.breached[i] != 0, cfg_.policy) && !pending_)
                    pending_ = decide_action(repo_, pht_, profiled_candidates(), serving_, depth_, cfg_.mem, mem_,
                                             cfg_.policy);
        }
    }

    EngineReport finish() {
        EngineReport r = rep_;
        if (r.tokens > 0) {
            r.throughput_tok_s = (double)r.tokens / r.decode_wall_s;
            r.perplexity = std::exp(-sum_logprob_ / (double)r.tokens);
            r.unchanged_fraction = unchanged_known_ ? (double)unchanged_ / (double)unchanged_known_ : 0.0;
            for (const auto& [m, per] : r.exit_counts)
                for (const auto& [l, c] : per) r.exit_table[m][l] = 100.0 * (double)c / (double)r.tokens;
        }
        if (!r.requests.empty()) {
            for (const auto& t : r.requests) {
                r.mean_ttft_s += t.ttft_s;
                r.mean_tpot_s += t.tokens ? t.tpot_sum_s / t.tokens : 0.0;
            }
            r.mean_ttft_s /= (double)r.requests.size();
            r.mean_tpot_s /= (double)r.requests.size();
        }
        r.pht = pht_;
        return r;
    }
};

}  // namespace eeserve
