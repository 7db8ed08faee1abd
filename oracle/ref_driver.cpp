// ref_driver.cpp — thin C driver over the UNMODIFIED reference headers
// (/root/reference/proj/include/eeserve, compiled in place by oracle/Makefile
// into oracle/_ref/libeeref.so).  TEST INFRASTRUCTURE ONLY: it lets the tests
// ask the reference itself for its exit rules, breach counter, profiler and
// scheduler decisions, and run its simulate() over traces our GPU produced.
// No reference source is copied into this repository.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "eeserve/config.hpp"
#include "eeserve/engine.hpp"
#include "eeserve/generator.hpp"
#include "eeserve/metrics.hpp"
#include "eeserve/policy.hpp"

using namespace eeserve;

namespace {
thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const ValidationError*>(&e)) return -1;
    if (dynamic_cast<const CapacityError*>(&e)) return -2;
    if (dynamic_cast<const DomainError*>(&e)) return -3;
    if (dynamic_cast<const StalenessError*>(&e)) return -4;
    return -9;
}

template <typename F>
int guard(F&& f) {
    try {
        return f();
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

ModelTokenRecord record_of(int n, const int* layers, const int* toks, const double* confs,
                           const double* logps, int final_tok) {
    ModelTokenRecord rec;
    rec.final_token_id = final_tok;
    for (int i = 0; i < n; ++i) rec.observations.push_back({layers[i], toks[i], confs[i], logps[i]});
    return rec;
}

int copy_out(const std::string& s, char* out, int cap) {
    if ((int)s.size() + 1 > cap) return -8;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return (int)s.size();
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// earliest_confident_obs (trace.hpp:69-76): returns the exit layer, token via out.
int ref_earliest_confident(int n, const int* layers, const int* toks, const double* confs,
                           const double* logps, double th, int* out_tok) {
    return guard([&] {
        const ModelTokenRecord rec = record_of(n, layers, toks, confs, logps, toks[n - 1]);
        const ExitObservation& o = earliest_confident_obs(rec, th);
        if (out_tok) *out_tok = o.token_id;
        return o.layer;
    });
}

// observation_for_depth (trace.hpp:86-97).
int ref_observation_for_depth(int n, const int* layers, const int* toks, const double* confs,
                              const double* logps, int depth, int* out_tok) {
    return guard([&] {
        const ModelTokenRecord rec = record_of(n, layers, toks, confs, logps, toks[n - 1]);
        const ExitObservation& o = observation_for_depth(rec, depth);
        if (out_tok) *out_tok = o.token_id;
        return o.layer;
    });
}

// observe_token (policy.hpp:147-156) over a breach sequence; triggers[i] = 1 when it fires.
int ref_observe_tokens(int n, const uint8_t* breached, int cbc_max, int window, uint8_t* triggers) {
    return guard([&] {
        PolicyConfig cfg;
        cfg.cbc_max = cbc_max;
        cfg.window = window;
        BreachTracker t;
        int fired = 0;
        for (int i = 0; i < n; ++i) {
            const bool f = observe_token(t, breached[i] != 0, cfg);
            triggers[i] = f ? 1 : 0;
            fired += f;
        }
        return fired;
    });
}

// choose_depth (pht.hpp:119-126) over a histogram keyed by exit layer.
int ref_choose_depth(int n_exits, const int* exits, const int64_t* counts, int num_layers,
                     double coverage) {
    return guard([&] {
        ModelSpec spec;
        spec.id = "m";
        spec.num_layers = num_layers;
        spec.exit_layers.assign(exits, exits + n_exits);
        ExitHistogram h;
        for (int i = 0; i < n_exits; ++i)
            if (counts[i] > 0) h.add(exits[i], counts[i]);
        return choose_depth(h, spec, coverage);
    });
}

// Run the reference simulate() over a JSONL trace; writes the report JSON
// (metrics_report_to_json) plus the final PHT into `out`.
int ref_simulate(const char* repo_json, const char* trace_jsonl, const char* mode, const char* policy_json,
                 const char* memory_json, char* out, int cap) {
    return guard([&] {
        const ModelRepository repo = load_repository(repo_json);
        const Trace trace = read_workload(trace_jsonl);
        const PolicyConfig pol = policy_config_from_json(Json::parse(policy_json));
        const MemoryConfig mem = memory_config_from_json(Json::parse(memory_json));
        const SimulationResult res = simulate(repo, trace, mem, pol, mode_spec_from_string(mode));
        Json j{{"report", metrics_report_to_json(res.report)}, {"pht", pht_to_json(res.pht)}};
        return copy_out(j.dump(), out, cap);
    });
}

// The reference's aggregate() (metrics.hpp:51-145) over an event log written
// by our engine (events.jsonl): the report it rebuilds, as JSON.
int ref_aggregate(const char* events_jsonl, char* out, int cap) {
    return guard([&] {
        const MetricsReport r = aggregate(read_event_log(events_jsonl));
        return copy_out(metrics_report_to_json(r).dump(), out, cap);
    });
}

// decide_action (policy.hpp:243-286) driven by a JSON description:
// {"repo": path, "pht": {id: {layer: count}}, "candidates": [...], "current": id,
//  "depth": d, "memory": {...}, "state": {id: depth}, "policy": {...}}
int ref_decide_action(const char* in_json, char* out, int cap) {
    return guard([&] {
        const Json in = Json::parse(in_json);
        const ModelRepository repo = load_repository(in.at("repo").get<std::string>());
        Pht pht;
        for (auto& [id, hist] : in.at("pht").items())
            for (auto& [layer, cnt] : hist.items())
                for (int64_t i = 0; i < cnt.get<int64_t>(); ++i)
                    record_token(pht, repo.at(id), std::stoi(layer), -0.1, 0.001);
        std::vector<std::string> cands = in.at("candidates").get<std::vector<std::string>>();
        MemoryState st;
        for (auto& [id, d] : in.at("state").items()) st.loaded_depth[id] = d.get<int>();
        const ActionPlan p = decide_action(repo, pht, cands, in.at("current").get<std::string>(),
                                           in.at("depth").get<int>(),
                                           memory_config_from_json(in.at("memory")), st,
                                           policy_config_from_json(in.at("policy")));
        Json j{{"kind", to_string(p.kind)}, {"model", p.model_id}, {"depth", p.serving_depth},
               {"evict", p.evict}, {"load_bytes", p.load_bytes}, {"cost_s", p.cost_s}};
        return copy_out(j.dump(), out, cap);
    });
}

// Generate a workload with the reference generator (generator.hpp:347) and
// write it as the reference JSONL trace format (trace.hpp:163-169).
int ref_generate_trace(const char* gen_json, const char* repo_json, const char* out_jsonl) {
    return guard([&] {
        const ModelRepository repo = load_repository(repo_json);
        const Trace t = generate_workload(load_generator_config(gen_json), repo);
        write_workload(t, out_jsonl);
        return (int)t.requests.size();
    });
}

}  // extern "C"
