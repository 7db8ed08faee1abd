// C3 serving run (BASELINE.json configs[2]): OPT-1.3B + OPT-2.7B shapes behind
// the host C++ engine (include/eeserve BatchedEngine, the drop-in for
// Simulator::run, engine.hpp:114-153) over CudaBackend and the C ABI: HELIOS
// mode with real-time profiling (evaluation cycles on both candidates, PHT,
// choose_depth), greedy layer loading from a pinned host tier, breach-driven
// switching, batch 256 with continuous batching over a paged KV pool.
// Prints one JSON line (bench.py attaches it as "secondary_c3").
//
//   serve_c3 [n_requests] [prompt_len] [tokens] [calib|drift]
//
// drift (default): the reference's drift workload shape (fixtures/gen_drift.json:
// alternating murky / easy segments with reference exit probabilities
// [0.3, 0.1, 0.6] / [0.92, 0.05, 0.03]).  The synthetic model decides a
// token's exit by its difficulty z(t) (synth.cuh: confident at head e iff
// z(t) <= cumulative coverage_e), so the teacher-forced input tokens are drawn
// per (request, position) from the z band of an exit sampled from the
// segment's law: murky segments breach at the greedy depth on the GPU and
// drive load-more / switch actions (test_engine.cpp:186-204).
// calib: uniformly drawn tokens (the calibration mixture).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "eeserve/engine.hpp"
#include "../paper_2504_10724_b200/csrc/synth.cuh"

using namespace eeserve;

static ModelSpec opt_shape(const std::string& id, int layers, std::vector<int> exits, int d, int heads, int ffn,
                           std::uint64_t seed, double thr, double t_layer) {
    ModelSpec s;
    s.id = id;
    s.num_layers = layers;
    s.exit_layers = std::move(exits);
    const std::int64_t bw = 2, vocab = 50272;
    s.per_layer_weight_bytes = (4LL * d * d + 2LL * d * ffn) * bw + 2LL * d * 4;
    s.base_weight_bytes = vocab * d * bw * (1 + (std::int64_t)s.exit_layers.size()) +
                          (std::int64_t)s.exit_layers.size() * d * 4;
    s.kv_bytes_per_token_per_layer = 2LL * d * bw;
    s.t_decode_per_layer_s = t_layer;
    s.t_prefill_per_layer_per_token_s = t_layer / 64.0;
    s.repo_metrics["throughput"] = thr;
    s.arch.d_model = d;
    s.arch.n_heads = heads;
    s.arch.n_kv_heads = heads;
    s.arch.d_ffn = ffn;
    s.arch.vocab = (int)vocab;
    s.arch.dtype = EEB_BF16;
    s.arch.seed = seed;
    validate_model_spec(s);
    return s;
}

// Wall time spent in each backend call, so the serving wall splits into GPU
// calls and the engine's own host work.
class TimedBackend final : public DecodeBackend {
public:
    explicit TimedBackend(DecodeBackend& inner) : in_(inner) {}
    double step_s = 0.0, prefill_s = 0.0, load_s = 0.0, other_s = 0.0;
    void register_model(const ModelSpec& spec, int max_slots, int max_seq_len) override {
        const auto t = now();
        in_.register_model(spec, max_slots, max_seq_len);
        other_s += since(t);
    }
    LoadResult load(const std::string& model, int depth) override {
        const auto t = now();
        const LoadResult r = in_.load(model, depth);
        load_s += since(t);
        return r;
    }
    double prefill(const std::string& model, int depth, const PrefillRows& rows) override {
        const auto t = now();
        const double r = in_.prefill(model, depth, rows);
        prefill_s += since(t);
        return r;
    }
    StepOutcome step(const std::string& model, int depth, TokenPolicy policy, double th,
                     const StepRows& rows) override {
        const auto t = now();
        StepOutcome r = in_.step(model, depth, policy, th, rows);
        step_s += since(t);
        return r;
    }
    void release(const std::string& model, int slot) override {
        const auto t = now();
        in_.release(model, slot);
        other_s += since(t);
    }

private:
    static std::chrono::steady_clock::time_point now() { return std::chrono::steady_clock::now(); }
    static double since(std::chrono::steady_clock::time_point t) {
        return std::chrono::duration<double>(now() - t).count();
    }
    DecodeBackend& in_;
};

int main(int argc, char** argv) {
    const int n_req = argc > 1 ? std::atoi(argv[1]) : 1024;
    const int prompt = argc > 2 ? std::atoi(argv[2]) : 128;
    const int tokens = argc > 3 ? std::atoi(argv[3]) : 64;
    const bool drift = argc > 4 ? std::string(argv[4]) != "calib" : true;
    ModelRepository repo;
    // public OPT dims: 1.3B L24 d2048 ffn 8192; 2.7B L32 d2560 ffn 10240; V 50272
    repo.models["opt-1.3b"] = opt_shape("opt-1.3b", 24, {6, 12, 24}, 2048, 32, 8192, 20260819, 2.0, 6e-5);
    repo.models["opt-2.7b"] = opt_shape("opt-2.7b", 32, {8, 16, 32}, 2560, 32, 10240, 20260820, 1.0, 8e-5);
    repo.metric_directions["throughput"] = MetricDirection::higher_better;

    EngineConfig cfg;
    cfg.mem.capacity_bytes = 40LL << 30;
    cfg.mem.reserve_bytes = 2LL << 30;
    cfg.mem.max_seq_len = prompt + tokens;
    cfg.mem.bandwidth_bytes_per_s = 8.4e9;  // modelled only where nothing is measured
    cfg.policy.k = 2;
    cfg.policy.n_eval_requests = 64;
    cfg.policy.ri = 512;
    cfg.policy.window = 100;
    cfg.policy.cbc_max = 50;
    cfg.mode = ModeSpec{Mode::helios, ""};
    cfg.max_batch = 256;
    cfg.max_seq_len = prompt + tokens;
    cfg.continuous = true;
    const int seg_len = 256;  // requests per drift segment
    if (drift) {
        // a token's difficulty is per model (its own seeded z): draw tokens
        // whose z lies in the sampled exit's band for BOTH candidates, so the
        // segment's law holds whichever model serves
        const std::uint64_t seed_a = repo.models["opt-1.3b"].arch.seed, seed_b = repo.models["opt-2.7b"].arch.seed;
        const std::vector<double> cum = {0.73, 0.777, 1.0};  // default coverage 73.0 / 4.7 / 22.3 %
        const double murky[3] = {0.3, 0.1, 0.6}, easy[3] = {0.92, 0.05, 0.03};
        // the vocabulary bucketed once by exit band (both models' z in the
        // band), so drawing a token is O(1) — rejection sampling for the
        // narrow middle band took ~100 us a token, host time that landed in
        // the serving wall
        const int vocab_all = repo.models["opt-1.3b"].arch.vocab;
        std::vector<std::vector<int32_t>> bands(3);
        for (int32_t t = 0; t < vocab_all; ++t) {
            const double za = eeb::synth::z_of(seed_a, t), zb = eeb::synth::z_of(seed_b, t);
            for (int e = 0; e < 3; ++e) {
                const double lo = (e == 0 ? 0.0 : cum[e - 1]) + 0.005, hi = cum[e] - 0.005;
                if (za >= lo && za < hi && zb >= lo && zb < hi) bands[e].push_back(t);
            }
        }
        for (const auto& b : bands)
            if (b.empty()) throw std::runtime_error("drift workload: an exit band holds no token of the vocabulary");
        cfg.token_fn = [=](std::int64_t rid, int pos, int /*vocab*/) -> int32_t {
            // easy, murky, easy, murky: the first evaluation sees an easy mix
            // (greedy depth at the first exit), the murky segments then breach
            const double* law = (rid / seg_len) % 2 == 0 ? easy : murky;
            const double u = (double)synthetic_token(0x5eedULL, rid, pos, 1 << 24) / (double)(1 << 24);
            const int e = u < law[0] ? 0 : (u < law[0] + law[1] ? 1 : 2);
            const auto& b = bands[e];
            return b[(size_t)synthetic_token(0x70c0ULL, rid, pos, (int)b.size())];
        };
    }

    const auto t0 = std::chrono::steady_clock::now();
    CudaBackend cuda_be(0, /*host_tier=*/true);
    cuda_be.set_kv_pages(64);  // pages for every slot BatchedEngine::slots_for sizes (max_batch_size)
    TimedBackend be(cuda_be);
    std::vector<RequestSpec> reqs;
    for (int i = 0; i < n_req; ++i) reqs.push_back({i, prompt, tokens});
    BatchedEngine eng(repo, be, cfg);
    eng.prepare();  // device pools sized from the memory model; both models staged in the pinned host tier
    const auto t1 = std::chrono::steady_clock::now();
    be.step_s = be.prefill_s = be.load_s = be.other_s = 0.0;  // (setup's calls are in setup_s)
    const EngineReport rep = eng.run(reqs);
    const auto t2 = std::chrono::steady_clock::now();
    const double setup_s = std::chrono::duration<double>(t1 - t0).count();
    const double run_s = std::chrono::duration<double>(t2 - t1).count();
    std::string exits = "{";
    for (const auto& [m, per] : rep.exit_table) {
        exits += (exits.size() > 1 ? ", \"" : "\"") + m + "\": {";
        bool first = true;
        for (const auto& [l, p] : per) {
            exits += (first ? "\"" : ", \"") + std::to_string(l) + "\": " + std::to_string(p);
            first = false;
        }
        exits += "}";
    }
    exits += "}";
    std::string hist = "[";
    for (size_t i = 0; i < rep.serving_history.size() && i < 12; ++i)
        hist += (i ? ", [\"" : "[\"") + rep.serving_history[i].first + "\", " +
                std::to_string(rep.serving_history[i].second) + "]";
    hist += "]";
    std::printf(
        "{\"workload\": \"C3: OPT-1.3B + OPT-2.7B shapes, HELIOS mode (eval cycles, PHT, choose_depth, greedy "
        "loads from a pinned host tier, breach switching), batch 256, continuous batching over a paged KV pool\", "
        "\"token_law\": \"%s\", \"slots\": {\"opt-1.3b\": %d, \"opt-2.7b\": %d}, "
        "\"requests\": %d, \"prompt_len\": %d, \"tokens_per_request\": %d, \"tokens\": %lld, \"steps\": %lld, "
        "\"decode_tokens_per_s\": %.1f, \"serving_tokens_per_s\": %.1f, \"wall_s\": %.3f, \"setup_s\": %.3f, "
        "\"mean_ttft_ms\": %.3f, \"mean_tpot_ms\": %.4f, \"achieved_batch\": %d, \"eval_cycles\": %lld, "
        "\"ld\": %lld, \"sw\": %lld, \"load_bytes\": %lld, \"load_s\": %.4f, \"load_gbs\": %.2f, \"prefill_s\": %.3f, "
        "\"perplexity\": %.6f, \"wall_split_s\": {\"step_calls\": %.3f, \"prefill_calls\": %.3f, \"load_calls\": %.3f, "
        "\"other_calls\": %.3f, \"engine_host\": %.3f}, \"exit_table_pct\": %s, \"serving_history\": %s}\n",
        drift ? "drift: easy/murky/easy/murky segments of 256 requests (gen_drift.json exit laws), tokens drawn by synthetic difficulty" : "calibration: uniform tokens",
        eng.slots("opt-1.3b"), eng.slots("opt-2.7b"), n_req, prompt, tokens, (long long)rep.tokens, (long long)rep.steps, rep.throughput_tok_s,
        rep.tokens / run_s, run_s, setup_s, rep.mean_ttft_s * 1e3, rep.mean_tpot_s * 1e3, rep.achieved_batch_size,
        (long long)rep.eval_cycles, (long long)rep.ld_count, (long long)rep.sw_count, (long long)rep.load_bytes,
        rep.load_s, rep.load_bytes / std::max(1e-9, rep.load_s) / 1e9, rep.prefill_s, rep.perplexity,
        be.step_s, be.prefill_s, be.load_s, be.other_s, run_s - be.step_s - be.prefill_s - be.load_s - be.other_s,
        exits.c_str(), hist.c_str());
    return 0;
}
