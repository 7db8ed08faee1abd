// GPU end-to-end check of the host C++ drop-in API (include/eeserve) over the
// C ABI: BatchedEngine (Simulator::run's control flow, engine.hpp:114-153)
// driving CudaBackend — real prefill (eeb_prefill), the greedy loader over a
// pinned host tier (eeb_load_layers_async / eeb_load_wait), batched decode
// steps and the profiler/scheduler (PHT, choose_depth, decide_action).
//
// The decision logic itself is pinned against the compiled reference on CPU
// (tests/cpp/test_host.cpp); this binary checks the integration on a B200.
#include <cmath>
#include <cstdio>
#include <string>

#include "eeserve/engine.hpp"
#include "../../paper_2504_10724_b200/csrc/synth.cuh"

using namespace eeserve;

static int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        ++g_checks;                                                       \
        if (!(c)) {                                                       \
            ++g_fail;                                                     \
            std::fprintf(stderr, "%s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
        }                                                                 \
    } while (0)

// A model descriptor whose byte counts follow its real bf16 dimensions.
static ModelSpec make_model(const std::string& id, int layers, std::vector<int> exits, int d, int heads, int ffn,
                            int vocab, std::uint64_t seed, double thr) {
    ModelSpec s;
    s.id = id;
    s.num_layers = layers;
    s.exit_layers = std::move(exits);
    const std::int64_t bw = 2;
    s.per_layer_weight_bytes = (4LL * d * d + 2LL * d * ffn) * bw + 2LL * d * 4;
    s.base_weight_bytes = (std::int64_t)vocab * d * bw * (1 + (std::int64_t)s.exit_layers.size()) +
                          (std::int64_t)s.exit_layers.size() * d * 4;
    s.kv_bytes_per_token_per_layer = 2LL * d * bw;
    s.t_decode_per_layer_s = 1e-4;
    s.t_prefill_per_layer_per_token_s = 1e-6;
    s.repo_metrics["throughput"] = thr;
    s.arch.d_model = d;
    s.arch.n_heads = heads;
    s.arch.n_kv_heads = heads;
    s.arch.d_ffn = ffn;
    s.arch.vocab = vocab;
    s.arch.dtype = EEB_BF16;
    s.arch.seed = seed;
    validate_model_spec(s);
    return s;
}

static ModelRepository make_repo() {
    ModelRepository r;
    r.models["small"] = make_model("small", 12, {6, 12}, 256, 4, 1024, 512, 7, 2.0);
    // a wider second model: switching regrows the shared workspace and KV
    // pools, which must invalidate the first model's captured graphs
    r.models["large"] = make_model("large", 16, {8, 16}, 512, 4, 2048, 768, 8, 1.0);
    r.metric_directions["throughput"] = MetricDirection::higher_better;
    return r;
}

static EngineConfig make_cfg(Mode mode, const std::string& model) {
    EngineConfig c;
    c.mem.capacity_bytes = 8LL << 30;
    c.mem.reserve_bytes = 1LL << 30;
    c.mem.max_seq_len = 64;
    c.mem.bandwidth_bytes_per_s = 8.4e9;
    c.policy.k = 2;
    c.policy.n_eval_requests = 16;
    c.policy.ri = 48;
    c.policy.window = 20;
    c.policy.cbc_max = 5;
    c.mode = ModeSpec{mode, model};
    c.max_batch = 16;
    c.max_seq_len = 64;
    return c;
}

static std::vector<RequestSpec> make_requests(int n) {
    std::vector<RequestSpec> v;
    for (int i = 0; i < n; ++i) v.push_back({i, 8 + (i % 5), 10 + (i % 3)});
    return v;
}

static void check_report(const EngineReport& rep, const std::vector<RequestSpec>& reqs) {
    std::int64_t want = 0;
    for (const auto& r : reqs) want += r.num_tokens;
    CHECK(rep.tokens == want);
    CHECK(rep.achieved_batch_size == 16);
    CHECK(rep.throughput_tok_s > 0.0);
    CHECK(std::isfinite(rep.perplexity) && rep.perplexity >= 1.0);
    double pct = 0.0;
    for (const auto& [m, per] : rep.exit_table)
        for (const auto& [l, p] : per) pct += p;
    CHECK(std::fabs(pct - 100.0) < 1e-6);
    CHECK(rep.requests.size() == reqs.size());
    for (const auto& t : rep.requests) CHECK(t.ttft_s > 0.0 && t.tokens > 0 && t.tpot_sum_s > 0.0);
    CHECK(rep.prefill_s > 0.0);
}

int main(int argc, char** argv) {
    const std::string events_path = argc > 1 ? argv[1] : "";
    const ModelRepository repo = make_repo();
    const auto reqs = make_requests(96);
    {  // HELIOS: eval cycles profile both candidates, replan, serve flat at the chosen depth
        CudaBackend be(0, /*host_tier=*/true);
        EngineConfig cfg = make_cfg(Mode::helios, "");
        cfg.record_events = !events_path.empty();
        BatchedEngine eng(repo, be, cfg);
        const EngineReport rep = eng.run(reqs);
        if (!events_path.empty()) {  // reference-format event log of a real GPU run (events.hpp)
            write_event_log(rep.events, events_path);
            std::printf("REPORT {\"throughput_tok_s\": %.17g, \"perplexity\": %.17g, \"mean_ttft_s\": %.17g, "
                        "\"mean_tpot_s\": %.17g, \"achieved_batch_size\": %d, \"ld\": %lld, \"sw\": %lld, "
                        "\"tokens\": %lld}\n",
                        rep.throughput_tok_s, rep.perplexity, rep.mean_ttft_s, rep.mean_tpot_s, rep.achieved_batch_size,
                        (long long)rep.ld_count, (long long)rep.sw_count, (long long)rep.tokens);
        }
        check_report(rep, reqs);
        CHECK(rep.eval_cycles >= 2);
        CHECK(rep.load_bytes > 0 && rep.load_s > 0.0);
        CHECK(rep.pht.has("small") && rep.pht.has("large"));
        bool flat_served = false;
        for (const auto& [m, d] : rep.serving_history) flat_served |= d < repo.at(m).num_layers;
        CHECK(flat_served);  // choose_depth picked a greedy prefix (biased heads: ~73% at the first exit)
        std::printf("helios: %lld tokens, %lld steps, %.0f tok/s, eval %lld, ld %lld, sw %lld, load %.3f ms "
                    "(%lld B, %.2f GB/s), prefill %.3f ms\n",
                    (long long)rep.tokens, (long long)rep.steps, rep.throughput_tok_s, (long long)rep.eval_cycles,
                    (long long)rep.ld_count, (long long)rep.sw_count, rep.load_s * 1e3, (long long)rep.load_bytes,
                    rep.load_bytes / std::max(1e-12, rep.load_s) / 1e9, rep.prefill_s * 1e3);
    }
    {  // drift: easy tokens while the candidates are profiled, then murky ones
       // (difficulty z(t) above every head's coverage) at the greedy depth —
       // the breach tracker must fire on real GPU verdicts and the engine apply
       // a load-more or switch at a request boundary (engine.hpp:381-385,
       // :301-323; the reference KAT is test_engine.cpp:186-204)
        CudaBackend be(0, /*host_tier=*/true);
        EngineConfig cfg = make_cfg(Mode::helios, "");
        const std::uint64_t seed = repo.at("small").arch.seed;
        cfg.token_fn = [seed](std::int64_t rid, int pos, int vocab) -> int32_t {
            const bool murky = rid >= 32;  // the first eval phase profiles 2 x 16 easy requests
            for (std::uint64_t k = 1;; ++k) {
                const int32_t t = synthetic_token(k * 0x9e3779b97f4a7c15ULL, rid, pos, vocab);
                const float z = eeb::synth::z_of(seed, t);
                if (murky ? z > 0.85f : z < 0.6f) return t;
            }
        };
        cfg.policy.ri = 1000;  // no reassessment after the first: only breaches move the plan
        BatchedEngine eng(repo, be, cfg);
        const EngineReport rep = eng.run(reqs);
        check_report(rep, reqs);
        CHECK(rep.ld_count + rep.sw_count >= 1);
        CHECK(rep.serving_history.size() >= 2);
        std::printf("drift: ld %lld, sw %lld, history", (long long)rep.ld_count, (long long)rep.sw_count);
        for (const auto& [m, d] : rep.serving_history) std::printf(" %s@%d", m.c_str(), d);
        std::printf("\n");
    }
    {  // drift with one candidate: no model to switch to, so the breach actions
       // deepen the serving model (load-more from the pinned host tier)
        CudaBackend be(0, /*host_tier=*/true);
        EngineConfig cfg = make_cfg(Mode::helios, "");
        cfg.policy.k = 1;
        const std::uint64_t seed = repo.at("small").arch.seed;
        cfg.token_fn = [seed](std::int64_t rid, int pos, int vocab) -> int32_t {
            const bool murky = rid >= 16;  // the first eval phase profiles 16 easy requests
            for (std::uint64_t k = 1;; ++k) {
                const int32_t t = synthetic_token(k * 0x9e3779b97f4a7c15ULL, rid, pos, vocab);
                const float z = eeb::synth::z_of(seed, t);
                if (murky ? z > 0.85f : z < 0.6f) return t;
            }
        };
        cfg.policy.ri = 1000;
        BatchedEngine eng(repo, be, cfg);
        const EngineReport rep = eng.run(reqs);
        check_report(rep, reqs);
        CHECK(rep.ld_count >= 1 && rep.sw_count == 0);
        std::printf("drift (k=1): ld %lld, sw %lld, history", (long long)rep.ld_count, (long long)rep.sw_count);
        for (const auto& [m, d] : rep.serving_history) std::printf(" %s@%d", m.c_str(), d);
        std::printf("\n");
    }
    {  // ee_single: introspective exits on the device; exit mixture near the calibrated 73/27
        CudaBackend be(0);
        BatchedEngine eng(repo, be, make_cfg(Mode::ee_single, "small"));
        const EngineReport rep = eng.run(reqs);
        check_report(rep, reqs);
        const double first = rep.exit_table.at("small").count(6) ? rep.exit_table.at("small").at(6) : 0.0;
        CHECK(first > 50.0 && first < 95.0);
        std::printf("ee_single: exit@6 %.1f%%, %.0f tok/s\n", first, rep.throughput_tok_s);
    }
    {  // continuous batching over a paged KV pool with exactly one page per slot:
       // every finished request must hand its page back before the next one is
       // admitted (else CapacityError); per-token decisions match static batching
        CudaBackend be_st(0);
        const EngineReport st = BatchedEngine(repo, be_st, make_cfg(Mode::ee_single, "small")).run(reqs);
        CudaBackend be(0);
        be.set_kv_pages(64, 16);
        EngineConfig cc = make_cfg(Mode::ee_single, "small");
        cc.continuous = true;
        const EngineReport rep = BatchedEngine(repo, be, cc).run(reqs);
        check_report(rep, reqs);
        CHECK(rep.steps < st.steps);
        // batch invariance: a row's result does not depend on its slot or on
        // the other rows of the step, so the exit tables agree exactly
        for (const auto& [l, p] : st.exit_table.at("small"))
            CHECK(std::fabs((rep.exit_table.at("small").count(l) ? rep.exit_table.at("small").at(l) : 0.0) - p) < 1e-9);
        std::printf("continuous+paged: %lld steps (static %lld), exit@6 %.1f%% (static %.1f%%)\n", (long long)rep.steps,
                    (long long)st.steps, rep.exit_table.at("small").count(6) ? rep.exit_table.at("small").at(6) : 0.0,
                    st.exit_table.at("small").count(6) ? st.exit_table.at("small").at(6) : 0.0);
    }
    {  // vanilla: every token at full depth
        CudaBackend be(0);
        BatchedEngine eng(repo, be, make_cfg(Mode::vanilla, "large"));
        const EngineReport rep = eng.run(reqs);
        check_report(rep, reqs);
        CHECK(rep.exit_table.at("large").size() == 1 && rep.exit_table.at("large").count(16) == 1);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
