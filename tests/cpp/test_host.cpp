// test_host.cpp — the host C++ drop-in API (include/eeserve) against the
// reference: its own known-answer tests re-hosted (Catch2 is absent, so a tiny
// CHECK shim stands in), randomized differential tests against the compiled
// reference (oracle/_ref/libeeref.so, test infrastructure), and the batched
// engine replaying reference traces at batch 1 against the reference
// simulate().  Fixtures: tests/golden/ (copies of /root/reference/proj/fixtures).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "eeserve/engine.hpp"

using namespace eeserve;
using Json = nlohmann::json;

// ---- shim -----------------------------------------------------------------------
static int g_fail = 0, g_checks = 0;
static std::vector<std::pair<std::string, std::function<void()>>>& registry() {
    static std::vector<std::pair<std::string, std::function<void()>>> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define TEST_CASE(name) static void name(); static Reg reg_##name(#name, name); static void name()
#define CHECK(c)                                                                            \
    do {                                                                                    \
        ++g_checks;                                                                         \
        if (!(c)) {                                                                         \
            ++g_fail;                                                                       \
            std::fprintf(stderr, "  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);             \
        }                                                                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                            \
    do {                                                                                    \
        ++g_checks;                                                                         \
        bool ok = false;                                                                    \
        try { (void)(expr); } catch (const T&) { ok = true; } catch (...) {}                \
        if (!ok) { ++g_fail; std::fprintf(stderr, "  FAIL %s:%d: %s !throws %s\n", __FILE__, __LINE__, #expr, #T); } \
    } while (0)
static bool approx(double a, double b, double rel = 1e-12) {
    return std::fabs(a - b) <= rel * std::max(std::fabs(a), std::fabs(b)) + 1e-300;
}

// ---- the compiled reference (oracle/_ref/libeeref.so) ---------------------------------
extern "C" {
int ref_earliest_confident(int, const int*, const int*, const double*, const double*, double, int*);
int ref_observation_for_depth(int, const int*, const int*, const double*, const double*, int, int*);
int ref_observe_tokens(int, const uint8_t*, int, int, uint8_t*);
int ref_choose_depth(int, const int*, const int64_t*, int, double);
int ref_simulate(const char*, const char*, const char*, const char*, const char*, char*, int);
int ref_decide_action(const char*, char*, int);
int ref_generate_trace(const char*, const char*, const char*);
int ref_aggregate(const char*, char*, int);
const char* ref_last_error();
}

static std::string g_golden;  // tests/golden
static std::string fx(const char* n) { return g_golden + "/" + n; }

// Fixture repositories rebuilt in code from the golden JSON.
static ModelRepository load_repo(const std::string& path) {
    std::ifstream in(path);
    Json j;
    in >> j;
    ModelRepository r;
    for (const auto& m : j.at("models")) {
        ModelSpec s;
        s.id = m.at("id");
        s.num_layers = m.at("num_layers");
        s.exit_layers = m.at("exit_layers").get<std::vector<int>>();
        s.base_weight_bytes = m.at("base_weight_bytes");
        s.per_layer_weight_bytes = m.at("per_layer_weight_bytes");
        s.kv_bytes_per_token_per_layer = m.at("kv_bytes_per_token_per_layer");
        s.t_decode_per_layer_s = m.at("t_decode_per_layer_s");
        s.t_prefill_per_layer_per_token_s = m.at("t_prefill_per_layer_per_token_s");
        if (m.contains("energy_per_layer_per_token_mwh")) s.energy_per_layer_per_token_mwh = m.at("energy_per_layer_per_token_mwh");
        for (auto& [k, v] : m.at("repo_metrics").items()) s.repo_metrics[k] = v.get<double>();
        validate_model_spec(s);
        r.models[s.id] = s;
    }
    for (auto& [k, v] : j.at("metric_directions").items())
        r.metric_directions[k] = v.get<std::string>() == "higher_better" ? MetricDirection::higher_better
                                                                        : MetricDirection::lower_better;
    return r;
}

static Trace load_trace(const std::string& path) {
    std::ifstream in(path);
    Trace t;
    std::string line;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        const Json j = Json::parse(line);
        TraceRequest r;
        r.request_id = j.at("request_id");
        r.arrival_time_s = j.at("arrival_time_s");
        r.prompt_len = j.at("prompt_len");
        for (const auto& tok : j.at("tokens")) {
            TokenRecord tr;
            for (auto& [mid, body] : tok.at("per_model").items()) {
                ModelTokenRecord rec;
                rec.final_token_id = body.at("final_token_id");
                for (const auto& o : body.at("observations"))
                    rec.observations.push_back({o.at("layer"), o.at("token_id"), o.at("confidence"), o.at("logprob")});
                tr.per_model[mid] = rec;
            }
            r.tokens.push_back(tr);
        }
        t.requests.push_back(r);
    }
    return t;
}

constexpr double T13 = 0.0009712509712509713;
constexpr double T67 = 0.0010451505016722408;

static Pht opt_pht(const ModelRepository& repo) {  // test_policy.cpp:17-31
    Pht pht;
    const ModelSpec& a = repo.at("opt-1.3b");
    const ModelSpec& b = repo.at("opt-6.7b");
    for (int i = 0; i < 73; ++i) record_token(pht, a, 6, -0.3852624007904164, 0.006);
    for (int i = 0; i < 5; ++i) record_token(pht, a, 12, -0.3852624007904164, 0.012);
    for (int i = 0; i < 22; ++i) record_token(pht, a, 24, -0.3852624007904164, 0.024);
    record_request(pht, a, 0.042);
    for (int i = 0; i < 72; ++i) record_token(pht, b, 9, -0.3987761199573, 0.009);
    for (int i = 0; i < 4; ++i) record_token(pht, b, 17, -0.3987761199573, 0.017);
    for (int i = 0; i < 24; ++i) record_token(pht, b, 32, -0.3987761199573, 0.032);
    record_request(pht, b, 0.069);
    return pht;
}

// ---- re-hosted reference KATs ------------------------------------------------------
TEST_CASE(trace_exit_rules_kat) {  // test_trace.cpp:39-63
    ModelTokenRecord rec;
    rec.final_token_id = 3;
    rec.observations = {{6, 1, 0.2, std::log(0.2)}, {12, 2, 0.6, std::log(0.6)}, {24, 3, 0.97, std::log(0.97)}};
    CHECK(earliest_confident_obs(rec, 0.5).layer == 12);
    CHECK(earliest_confident_obs(rec, 0.7).layer == 24);
    CHECK(earliest_confident_obs(rec, 0.1).layer == 6);
    CHECK(earliest_confident_obs(rec, 0.99).layer == 24);
    CHECK(earliest_confident_obs(rec, 0.5).token_id == 2);
    TokenRecord t;
    t.per_model["opt-1.3b"] = rec;
    CHECK(earliest_confident_exit(t, "opt-1.3b", 0.5) == 12);
    CHECK_THROWS_AS(t.for_model("opt-13b"), DomainError);
    CHECK(exit_index({6, 12, 24}, 12) == 1);
    CHECK_THROWS_AS(exit_index({6, 12, 24}, 7), DomainError);
    ModelTokenRecord r2;
    r2.final_token_id = 9;
    r2.observations = {{6, 4, 0.3, -1.2}, {12, 7, 0.8, -0.22}, {24, 9, 0.99, -0.01}};
    CHECK(observation_for_depth(r2, 12).token_id == 7);
    CHECK(observation_for_depth(r2, 17).layer == 12);
    CHECK(observation_for_depth(r2, 30).layer == 24);
    CHECK_THROWS_AS(observation_for_depth(r2, 3), DomainError);
    CHECK(r2.at_layer(24).token_id == 9);
    CHECK_THROWS_AS(r2.at_layer(7), DomainError);
}

TEST_CASE(pht_kats) {  // test_pht.cpp:11-91
    ExitHistogram h;
    h.add(6, 73);
    h.add(12, 5);
    h.add(24, 22);
    CHECK(h.total == 100);
    CHECK(h.frac(6) == 0.73);
    CHECK(h.frac(9) == 0.0);
    CHECK(h.cum_frac(12) == 0.78);
    CHECK(h.cum_frac(24) == 1.0);
    CHECK(h.cum_frac(5) == 0.0);
    CHECK(point_mass(12).frac(12) == 1.0);
    CHECK_THROWS_AS(ExitHistogram{}.frac(6), StalenessError);
    const ModelRepository repo = load_repo(fx("repo_opt.json"));
    const ModelSpec& m13 = repo.at("opt-1.3b");
    CHECK(choose_depth(h, m13, 0.70) == 6);
    CHECK(choose_depth(h, m13, 0.73) == 6);
    CHECK(choose_depth(h, m13, 0.74) == 12);
    CHECK(choose_depth(h, m13, 0.78) == 12);
    CHECK(choose_depth(h, m13, 0.79) == 24);
    CHECK(choose_depth(h, m13, 1.0) == 24);
    CHECK_THROWS_AS(choose_depth(h, m13, 0.0), DomainError);
    CHECK_THROWS_AS(choose_depth(h, m13, 1.5), DomainError);
    CHECK_THROWS_AS(choose_depth(ExitHistogram{}, m13, 0.7), DomainError);
    Pht pht;
    record_token(pht, m13, 6, -0.385262400790, 0.006);
    record_token(pht, m13, 24, -0.398776119957, 0.024);
    record_request(pht, m13, 0.042);
    record_request(pht, m13, 0.044);
    const PhtEntry& e = pht.entry_of("opt-1.3b");
    CHECK(e.token_count == 2);
    CHECK(approx(e.measured_tpot_s(), 0.015));
    CHECK(approx(e.measured_ttft_s(), 0.043));
    CHECK(approx(*e.perplexity(), 1.4799662159, 1e-9));
    CHECK(!perplexity(pht, "opt-6.7b").has_value());
    CHECK_THROWS_AS(record_token(pht, m13, 7, -0.1, 0.007), DomainError);
    pht.reset("opt-1.3b");
    CHECK(!pht.has("opt-1.3b"));
    CHECK_THROWS_AS(pht.entry_of("opt-1.3b"), StalenessError);
    // batched form == per-token form
    Pht a, b;
    record_step(a, m13, {3, 1, 2}, -1.5, 0.01);
    for (int l : {6, 6, 6, 12, 24, 24}) record_token(b, m13, l, -0.25, 0.01);
    CHECK(a.entry_of("opt-1.3b").exit_hist.counts == b.entry_of("opt-1.3b").exit_hist.counts);
    CHECK(approx(a.entry_of("opt-1.3b").sum_neg_logprob, b.entry_of("opt-1.3b").sum_neg_logprob));
    CHECK(approx(a.entry_of("opt-1.3b").tpot_sum_s, b.entry_of("opt-1.3b").tpot_sum_s));
}

TEST_CASE(breach_tracker_kat) {  // test_policy.cpp:111-131
    PolicyConfig cfg;
    BreachTracker t;
    for (int i = 0; i < 50; ++i) CHECK(!observe_token(t, true, cfg));
    CHECK(observe_token(t, true, cfg));
    CHECK(t.cbc == 0 && t.tokens_in_window == 0);
    for (int i = 0; i < 50; ++i) CHECK(!observe_token(t, true, cfg));
    for (int i = 0; i < 50; ++i) CHECK(!observe_token(t, false, cfg));
    CHECK(t.tokens_in_window == 0);
    for (int i = 0; i < 50; ++i) CHECK(!observe_token(t, true, cfg));
    CHECK(observe_token(t, true, cfg));
    BreachTracker u;
    for (int i = 0; i < 1000; ++i) CHECK(!observe_token(u, i % 2 == 0, cfg));
}

TEST_CASE(latency_and_decide_action_kats) {  // test_policy.cpp:133-244
    const ModelRepository repo = load_repo(fx("repo_opt.json"));
    const ModelSpec& m13 = repo.at("opt-1.3b");
    const ModelSpec& m67 = repo.at("opt-6.7b");
    ExitHistogram h;
    h.add(6, 73);
    h.add(12, 5);
    h.add(24, 22);
    CHECK(approx(expected_token_latency(h, m13, 24), 10.26 * T13));
    CHECK(approx(expected_token_latency(h, m13, 12), 7.62 * T13));
    CHECK(approx(expected_token_latency(h, m13, 6), 6 * T13));
    CHECK(approx(expected_token_latency(point_mass(9), m67, 9), 0.0094063545150501672));
    CHECK(approx(expected_token_energy(h, m13, 6), 6 * 0.48562548562548564));
    const Pht pht = opt_pht(repo);
    const std::vector<std::string> cands = {"opt-1.3b", "opt-6.7b"};
    const MemoryConfig mem{40'000'000'000, 1'000'000'000, 256, 8.4e9};
    const PolicyConfig cfg;
    {
        MemoryState st;
        st.loaded_depth = {{"opt-1.3b", 6}, {"opt-6.7b", 9}};
        const ActionPlan p = decide_action(repo, pht, cands, "opt-1.3b", 6, mem, st, cfg);
        CHECK(p.kind == ActionKind::switch_model && p.model_id == "opt-6.7b" && p.serving_depth == 9);
        CHECK(p.load_bytes == 0 && p.evict.empty());
        CHECK(approx(p.cost_s, (9 * T67) / 804));
    }
    {
        MemoryState st;
        st.loaded_depth = {{"opt-1.3b", 6}};
        const ActionPlan p = decide_action(repo, pht, cands, "opt-1.3b", 6, mem, st, cfg);
        CHECK(p.kind == ActionKind::load_more && p.serving_depth == 12);
        CHECK(p.load_bytes == 6 * 187'222'222LL);
        CHECK(approx(p.cost_s, ((6.0 * 187'222'222) / 8.4e9) / 1000.0 + (7.62 * T13) / 1450.0));
    }
    {
        MemoryState st;
        st.loaded_depth = {{"opt-1.3b", 24}};
        const ActionPlan p = decide_action(repo, pht, cands, "opt-1.3b", 24, mem, st, cfg);
        CHECK(p.kind == ActionKind::switch_model && p.serving_depth == 9 && p.load_bytes == 7'250'000'000LL);
        CHECK(approx(p.cost_s, (7.25e9 / 8.4e9) / 1000.0 + (9 * T67) / 715.0));
    }
    {
        const MemoryConfig tight{8'000'000'000, 0, 256, 8.4e9};
        MemoryState st;
        st.loaded_depth = {{"opt-1.3b", 24}};
        const ActionPlan p = decide_action(repo, pht, cands, "opt-1.3b", 24, tight, st, cfg);
        CHECK(p.kind == ActionKind::switch_model && p.evict == std::vector<std::string>{"opt-1.3b"});
    }
    {
        const MemoryConfig tiny{2'000'000'000, 0, 256, 8.4e9};
        MemoryState st;
        st.loaded_depth = {{"opt-1.3b", 6}};
        const ActionPlan p = decide_action(repo, pht, cands, "opt-1.3b", 6, tiny, st, cfg);
        CHECK(p.kind == ActionKind::stay && p.serving_depth == 6 && p.cost_s == 0.0);
    }
    {
        Pht partial;
        record_token(partial, m13, 6, -0.4, 0.006);
        MemoryState st;
        st.loaded_depth = {{"opt-1.3b", 6}};
        CHECK_THROWS_AS(decide_action(repo, partial, cands, "opt-1.3b", 6, mem, st, cfg), StalenessError);
    }
    const ReplanResult plan = replan_after_eval(repo, pht, cands, cfg, mem);
    CHECK(plan.serving_model == "opt-1.3b" && plan.serving_depth == 6);
    CHECK(plan.residency.size() == 2 && plan.residency[1] == std::make_pair(std::string("opt-6.7b"), 9));
    CHECK(best_model(repo, pht, cands, Slo::accuracy, 0.70) == "opt-1.3b");
}

TEST_CASE(memory_model_kats) {  // test_memory_model.cpp:11-80
    const ModelRepository repo = load_repo(fx("repo_large.json"));
    const MemoryConfig cfg{160'000'000'000, 0, 1000, 8.4e9};
    MemoryState st;
    apply_load(st, repo, cfg, "codellama-34b", 48);
    CHECK(weights_loaded_bytes(st, repo) == 63'000'000'000LL);
    CHECK_THROWS_AS(apply_load(st, repo, cfg, "llama2-70b", 80), CapacityError);
    CHECK(st.depth_of("llama2-70b") == 0);
    apply_load(st, repo, cfg, "codellama-34b", 12);
    apply_load(st, repo, cfg, "llama2-70b", 10);
    CHECK(weights_loaded_bytes(st, repo) == 42'000'000'000LL);
    CHECK(kv_budget_bytes(cfg, st, repo) == 118'000'000'000LL);
    const ModelSpec& cl = repo.at("codellama-34b");
    const MemoryConfig c80{80'000'000'000, 650'000'000, 1000, 8.4e9};
    MemoryState full, part;
    apply_load(full, repo, c80, "codellama-34b", 48);
    apply_load(part, repo, c80, "codellama-34b", 12);
    const int bf = max_batch_size(cl, 48, kv_budget_bytes(c80, full, repo), 1000);
    const int bp = max_batch_size(cl, 12, kv_budget_bytes(c80, part, repo), 1000);
    CHECK(bf == 50);
    CHECK(bp == 757);  // the 15.14x batch growth
    const ModelRepository ro = load_repo(fx("repo_opt.json"));
    const ModelSpec& m67 = ro.at("opt-6.7b");
    CHECK(load_delta_bytes(m67, 0, 9) == 7'250'000'000LL);
    CHECK(load_delta_bytes(m67, 32, 9) == 0);
    const MemoryConfig m40{40'000'000'000, 1'000'000'000, 256, 8.4e9};
    CHECK(load_seconds(8'400'000'000, m40) == 1.0);
}

// ---- differential tests against the compiled reference ----------------------------------
TEST_CASE(exit_rules_match_reference_randomized) {
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    for (int it = 0; it < 20000; ++it) {
        const int n = 1 + (int)(rng() % 5);
        std::vector<int> layers, toks;
        std::vector<double> conf, logp;
        int l = 0;
        for (int i = 0; i < n; ++i) {
            l += 1 + (int)(rng() % 8);
            layers.push_back(l);
            toks.push_back((int)(rng() % 50));
            const double c = (rng() % 10 == 0) ? 0.7 : U(rng);  // exact-threshold ties on purpose
            conf.push_back(c);
            logp.push_back(std::log(std::max(c, 1e-6)));
        }
        ModelTokenRecord rec;
        rec.final_token_id = toks.back();
        for (int i = 0; i < n; ++i) rec.observations.push_back({layers[i], toks[i], conf[i], logp[i]});
        const double th = (rng() % 4 == 0) ? 0.7 : U(rng);
        int rt = -1;
        const int rl = ref_earliest_confident(n, layers.data(), toks.data(), conf.data(), logp.data(), th, &rt);
        CHECK(rl == earliest_confident_obs(rec, th).layer);
        CHECK(rt == earliest_confident_obs(rec, th).token_id);
        const int depth = (int)(rng() % (l + 3));
        int ft = -1;
        const int fl = ref_observation_for_depth(n, layers.data(), toks.data(), conf.data(), logp.data(), depth, &ft);
        if (fl == -3) {
            CHECK_THROWS_AS(observation_for_depth(rec, depth), DomainError);
        } else {
            CHECK(fl == observation_for_depth(rec, depth).layer);
            CHECK(ft == observation_for_depth(rec, depth).token_id);
        }
    }
}

TEST_CASE(breach_and_depth_match_reference_randomized) {
    std::mt19937_64 rng(11);
    for (int it = 0; it < 200; ++it) {
        const int window = 1 + (int)(rng() % 150);
        const int cbc = 1 + (int)(rng() % window);
        const double p = (double)(rng() % 100) / 100.0;
        std::vector<uint8_t> br(3000), trig(3000);
        for (auto& b : br) b = (rng() % 1000) < p * 1000 ? 1 : 0;
        ref_observe_tokens((int)br.size(), br.data(), cbc, window, trig.data());
        PolicyConfig cfg;
        cfg.cbc_max = cbc;
        cfg.window = window;
        BreachTracker t;
        for (size_t i = 0; i < br.size(); ++i) CHECK((uint8_t)observe_token(t, br[i] != 0, cfg) == trig[i]);
        std::vector<int> exits = {6, 12, 18, 24};
        std::vector<int64_t> counts = {(int64_t)(rng() % 100), (int64_t)(rng() % 10), (int64_t)(rng() % 10),
                                       (int64_t)(rng() % 40) + 1};
        const double cov = (double)(1 + rng() % 100) / 100.0;
        ModelSpec s;
        s.id = "m";
        s.num_layers = 24;
        s.exit_layers = exits;
        ExitHistogram h;
        for (int i = 0; i < 4; ++i)
            if (counts[i]) h.add(exits[i], counts[i]);
        CHECK(ref_choose_depth(4, exits.data(), counts.data(), 24, cov) == choose_depth(h, s, cov));
    }
}

TEST_CASE(decide_action_matches_reference_randomized) {
    const std::string path = fx("repo_opt.json");
    const ModelRepository repo = load_repo(path);
    std::mt19937_64 rng(5);
    const std::vector<int> d13 = {6, 12, 24}, d67 = {9, 17, 32};
    char buf[4096];
    for (int it = 0; it < 300; ++it) {
        Json pj;
        Pht pht;
        for (const auto& [id, ex] : {std::make_pair(std::string("opt-1.3b"), d13), std::make_pair(std::string("opt-6.7b"), d67)}) {
            for (int l : ex) {
                const int c = (int)(rng() % 50) + (l == ex.back() ? 1 : 0);
                pj[id][std::to_string(l)] = c;
                for (int k = 0; k < c; ++k) record_token(pht, repo.at(id), l, -0.1, 0.001);
            }
        }
        const std::string cur = rng() % 2 ? "opt-1.3b" : "opt-6.7b";
        const std::vector<int>& cex = cur == "opt-1.3b" ? d13 : d67;
        const int depth = cex[rng() % cex.size()];
        MemoryState st;
        Json sj = Json::object();
        st.loaded_depth[cur] = depth;
        sj[cur] = depth;
        if (rng() % 2) {
            const std::string o = cur == "opt-1.3b" ? "opt-6.7b" : "opt-1.3b";
            const std::vector<int>& oex = o == "opt-1.3b" ? d13 : d67;
            st.loaded_depth[o] = oex[rng() % oex.size()];
            sj[o] = st.loaded_depth[o];
        }
        const int64_t caps[] = {8'000'000'000, 20'000'000'000, 40'000'000'000, 80'000'000'000};
        const MemoryConfig mem{caps[rng() % 4], (int64_t)(rng() % 2) * 1'000'000'000, 256, 8.4e9};
        PolicyConfig pol;
        pol.slo = (Slo)(rng() % 4);
        pol.horizon_tokens = 100 + (int)(rng() % 2000);
        pol.coverage_target = 0.5 + 0.05 * (double)(rng() % 10);
        Json in{{"repo", path}, {"pht", pj}, {"candidates", {"opt-1.3b", "opt-6.7b"}}, {"current", cur},
                {"depth", depth},
                {"memory", {{"capacity_bytes", mem.capacity_bytes}, {"reserve_bytes", mem.reserve_bytes},
                            {"max_seq_len", mem.max_seq_len}, {"bandwidth_bytes_per_s", mem.bandwidth_bytes_per_s}}},
                {"state", sj},
                {"policy", {{"slo", to_string(pol.slo)}, {"horizon_tokens", pol.horizon_tokens},
                            {"coverage_target", pol.coverage_target}}}};
        const int rc = ref_decide_action(in.dump().c_str(), buf, sizeof buf);
        bool threw = false;
        ActionPlan mine;
        try {
            mine = decide_action(repo, pht, {"opt-1.3b", "opt-6.7b"}, cur, depth, mem, st, pol);
        } catch (const std::exception&) {
            threw = true;
        }
        CHECK(threw == (rc < 0));
        if (rc < 0 || threw) continue;
        const Json r = Json::parse(buf);
        CHECK(r.at("kind").get<std::string>() == to_string(mine.kind));
        CHECK(r.at("model").get<std::string>() == mine.model_id);
        CHECK(r.at("depth").get<int>() == mine.serving_depth);
        CHECK(r.at("load_bytes").get<int64_t>() == mine.load_bytes);
        CHECK(r.at("cost_s").get<double>() == mine.cost_s);  // bit-identical arithmetic
        CHECK(r.at("evict").get<std::vector<std::string>>() == mine.evict);
    }
}

// ---- the batched engine replaying reference traces at batch 1 ---------------------------
static void engine_matches_reference(const std::string& trace_path, const std::string& mode_str, Mode mode,
                                     const std::string& model, int k, bool continuous = false, int ri = 150,
                                     int window = 100, int cbc_max = 50) {
    const ModelRepository repo = load_repo(fx("repo_opt.json"));
    const Trace trace = load_trace(trace_path);
    const MemoryConfig mem{40'000'000'000, 1'000'000'000, 256, 8.4e9};
    PolicyConfig pol;
    pol.k = k;
    pol.n_eval_requests = 5;
    pol.ri = ri;
    pol.window = window;
    pol.cbc_max = cbc_max;
    const std::string pj =
        Json{{"k", k}, {"n_eval_requests", 5}, {"ri", ri}, {"window", window}, {"cbc_max", cbc_max}}.dump();
    const std::string mj = Json{{"capacity_bytes", mem.capacity_bytes}, {"reserve_bytes", mem.reserve_bytes},
                                {"max_seq_len", 256}, {"bandwidth_bytes_per_s", 8.4e9}}.dump();
    std::vector<char> buf(1 << 24);
    const int rc = ref_simulate(fx("repo_opt.json").c_str(), trace_path.c_str(), mode_str.c_str(), pj.c_str(),
                                mj.c_str(), buf.data(), (int)buf.size());
    CHECK(rc > 0);
    if (rc <= 0) {
        std::fprintf(stderr, "  ref_simulate: %s\n", ref_last_error());
        return;
    }
    const Json ref = Json::parse(buf.data());
    TraceBackend be(trace);
    EngineConfig cfg;
    cfg.mem = mem;
    cfg.policy = pol;
    cfg.mode = ModeSpec{mode, model};
    cfg.max_batch = 1;
    cfg.prefill = false;
    cfg.record_events = true;
    cfg.continuous = continuous;
    BatchedEngine eng(repo, be, cfg);
    std::vector<RequestSpec> reqs;
    for (const auto& r : trace.requests) reqs.push_back({r.request_id, r.prompt_len, r.num_tokens()});
    const EngineReport rep = eng.run(reqs);
    // Event-log parity: the reference's aggregate() over OUR event log must
    // rebuild the reference simulate()'s own report (metrics.hpp:51-145).
    {
        const std::string log = "/tmp/eeserve_engine_events.jsonl";
        write_event_log(rep.events, log);
        std::vector<char> ab(1 << 24);
        const int arc = ref_aggregate(log.c_str(), ab.data(), (int)ab.size());
        CHECK(arc > 0);
        if (arc > 0) {
            const Json agg = Json::parse(ab.data());
            const Json& a1 = agg.at("aggregates");
            const Json& a0 = ref.at("report").at("aggregates");
            for (const char* k : {"throughput_tok_s", "mean_ttft_s", "mean_tpot_s", "perplexity",
                                  "energy_mwh_per_prompt", "unchanged_fraction"})
                CHECK(approx(a1.at(k).get<double>(), a0.at(k).get<double>(), 1e-9));
            CHECK(a1.at("achieved_batch_size") == a0.at("achieved_batch_size"));
            CHECK(agg.at("action_counts") == ref.at("report").at("action_counts"));
            CHECK(agg.at("exit_table").size() == ref.at("report").at("exit_table").size());
            for (auto& [m, per] : ref.at("report").at("exit_table").items())
                for (auto& [layer, pct] : per.items())
                    CHECK(approx(agg.at("exit_table").at(m).at(layer).get<double>(), pct.get<double>(), 1e-12));
            CHECK(agg.at("per_request").size() == ref.at("report").at("per_request").size());
            CHECK(approx(a1.at("mean_ttft_s").get<double>(), rep.mean_ttft_s, 1e-9));
        }
    }
    const Json& et = ref.at("report").at("exit_table");
    int rows = 0;
    for (auto& [m, per] : et.items())
        for (auto& [layer, pct] : per.items()) {
            ++rows;
            CHECK(approx(rep.exit_table.at(m).at(std::stoi(layer)), pct.get<double>(), 1e-12));
        }
    size_t mine_rows = 0;
    for (const auto& [m, per] : rep.exit_table) mine_rows += per.size();
    CHECK((size_t)rows == mine_rows);
    const Json& ag = ref.at("report").at("aggregates");
    CHECK(approx(rep.perplexity, ag.at("perplexity").get<double>(), 1e-12));
    CHECK(approx(rep.throughput_tok_s, ag.at("throughput_tok_s").get<double>(), 1e-9));
    CHECK(rep.ld_count == ref.at("report").at("action_counts").at("ld").get<int64_t>());
    CHECK(rep.sw_count == ref.at("report").at("action_counts").at("sw").get<int64_t>());
    for (auto& [m, e] : ref.at("pht").items()) {
        if (e.at("token_count").get<int64_t>() == 0) continue;
        CHECK(rep.pht.has(m));
        if (!rep.pht.has(m)) continue;
        CHECK(rep.pht.entry_of(m).token_count == e.at("token_count").get<int64_t>());
        CHECK(approx(*rep.pht.entry_of(m).perplexity(), e.at("perplexity").get<double>(), 1e-12));
    }
}

// Batched (width 4) run through the trace backend: the reference's aggregate()
// over the engine's event log rebuilds the engine's own report, with a
// decode step of 4 rows counted once (same t_s, metrics.hpp:85-93).
TEST_CASE(event_log_aggregates_to_engine_report_at_batch_4) {
    const std::string gen = "/tmp/eeserve_gen_small_b4.jsonl";
    CHECK(ref_generate_trace(fx("gen_small.json").c_str(), fx("repo_opt.json").c_str(), gen.c_str()) == 10);
    const ModelRepository repo = load_repo(fx("repo_opt.json"));
    const Trace trace = load_trace(gen);
    TraceBackend be(trace);
    EngineConfig cfg;
    cfg.mem = MemoryConfig{40'000'000'000, 1'000'000'000, 256, 8.4e9};
    cfg.policy.k = 2;
    cfg.mode = ModeSpec{Mode::helios, ""};
    cfg.max_batch = 4;
    cfg.prefill = false;
    cfg.record_events = true;
    BatchedEngine eng(repo, be, cfg);
    std::vector<RequestSpec> reqs;
    for (const auto& r : trace.requests) reqs.push_back({r.request_id, r.prompt_len, r.num_tokens()});
    const EngineReport rep = eng.run(reqs);
    const std::string log = "/tmp/eeserve_engine_events_b4.jsonl";
    write_event_log(rep.events, log);
    std::vector<char> ab(1 << 24);
    CHECK(ref_aggregate(log.c_str(), ab.data(), (int)ab.size()) > 0);
    const Json agg = Json::parse(ab.data());
    const Json& a = agg.at("aggregates");
    CHECK(approx(a.at("throughput_tok_s").get<double>(), rep.throughput_tok_s, 1e-9));
    CHECK(approx(a.at("perplexity").get<double>(), rep.perplexity, 1e-12));
    CHECK(approx(a.at("mean_ttft_s").get<double>(), rep.mean_ttft_s, 1e-9));
    CHECK(approx(a.at("mean_tpot_s").get<double>(), rep.mean_tpot_s, 1e-9));
    CHECK(a.at("achieved_batch_size").get<int>() == rep.achieved_batch_size);
    CHECK(rep.achieved_batch_size == 4);
    CHECK(agg.at("action_counts").at("ld").get<int64_t>() == rep.ld_count);
    CHECK(agg.at("action_counts").at("sw").get<int64_t>() == rep.sw_count);
    for (const auto& [m, per] : rep.exit_table)
        for (const auto& [l, pct] : per)
            CHECK(approx(agg.at("exit_table").at(m).at(std::to_string(l)).get<double>(), pct, 1e-12));
    CHECK(agg.at("per_request").size() == reqs.size());
}

// Breach actions: the drift workload (fixtures/gen_drift.json) at the
// reference's drift policy (exp_drift.json: k 1, ri 300, window 100,
// cbc_max 50) and at a tighter breach window that also switches models.
TEST_CASE(engine_matches_reference_under_breaches) {
    const std::string gen = "/tmp/eeserve_gen_drift.jsonl";
    CHECK(ref_generate_trace(fx("gen_drift.json").c_str(), fx("repo_opt.json").c_str(), gen.c_str()) == 3000);
    engine_matches_reference(gen, "helios", Mode::helios, "", 1, false, 300, 100, 50);
    engine_matches_reference(gen, "helios", Mode::helios, "", 1, false, 40, 20, 5);
}

TEST_CASE(engine_replays_reference_traces_at_batch_1) {
    const std::string gen = "/tmp/eeserve_gen_small.jsonl";
    CHECK(ref_generate_trace(fx("gen_small.json").c_str(), fx("repo_opt.json").c_str(), gen.c_str()) == 10);
    engine_matches_reference(gen, "vanilla:opt-1.3b", Mode::vanilla, "opt-1.3b", 2);
    engine_matches_reference(gen, "ee_single:opt-1.3b", Mode::ee_single, "opt-1.3b", 2);
    engine_matches_reference(gen, "ee_single:opt-6.7b", Mode::ee_single, "opt-6.7b", 2);
    engine_matches_reference(gen, "helios", Mode::helios, "", 2);
    engine_matches_reference(fx("eval_quality.jsonl"), "helios", Mode::helios, "", 2);  // PHT 1.47 / 1.49
}

// Continuous batching (EngineConfig::continuous): at width 1 it is the
// reference loop (same report, same event log through the reference
// aggregate()); at width 4 the teacher-forced traces give every token the same
// observation however requests interleave, so the exit table, perplexity and
// token count equal the reference's, with decode steps 4 rows wide and the
// event log still aggregating to the engine's own report.
TEST_CASE(continuous_batching_matches_reference) {
    const std::string gen = "/tmp/eeserve_gen_small_cb.jsonl";
    CHECK(ref_generate_trace(fx("gen_small.json").c_str(), fx("repo_opt.json").c_str(), gen.c_str()) == 10);
    engine_matches_reference(gen, "ee_single:opt-1.3b", Mode::ee_single, "opt-1.3b", 2, true);
    engine_matches_reference(gen, "helios", Mode::helios, "", 2, true);
    const ModelRepository repo = load_repo(fx("repo_opt.json"));
    const Trace trace = load_trace(gen);
    std::vector<RequestSpec> reqs;
    for (const auto& r : trace.requests) reqs.push_back({r.request_id, r.prompt_len, r.num_tokens()});
    auto run = [&](int width, bool continuous) {
        TraceBackend be(trace);
        EngineConfig cfg;
        cfg.mem = MemoryConfig{40'000'000'000, 1'000'000'000, 256, 8.4e9};
        cfg.mode = ModeSpec{Mode::ee_single, "opt-1.3b"};
        cfg.max_batch = width;
        cfg.prefill = false;
        cfg.record_events = true;
        cfg.continuous = continuous;
        BatchedEngine eng(repo, be, cfg);
        return eng.run(reqs);
    };
    const EngineReport one = run(1, false), cb = run(4, true), st = run(4, false);
    CHECK(cb.tokens == one.tokens);
    CHECK(approx(cb.perplexity, one.perplexity, 1e-12));
    for (const auto& [m, per] : one.exit_table)
        for (const auto& [l, pct] : per) CHECK(approx(cb.exit_table.at(m).at(l), pct, 1e-12));
    CHECK(cb.achieved_batch_size == 4);
    CHECK(cb.steps < one.steps);
    CHECK(cb.steps <= st.steps);  // a freed slot is refilled at once: never more steps than static batches
    CHECK(cb.requests.size() == reqs.size());
    const std::string log = "/tmp/eeserve_engine_events_cb.jsonl";
    write_event_log(cb.events, log);
    std::vector<char> ab(1 << 24);
    CHECK(ref_aggregate(log.c_str(), ab.data(), (int)ab.size()) > 0);
    const Json agg = Json::parse(ab.data());
    const Json& a = agg.at("aggregates");
    CHECK(approx(a.at("throughput_tok_s").get<double>(), cb.throughput_tok_s, 1e-9));
    CHECK(approx(a.at("perplexity").get<double>(), cb.perplexity, 1e-12));
    CHECK(approx(a.at("mean_ttft_s").get<double>(), cb.mean_ttft_s, 1e-9));
    CHECK(a.at("achieved_batch_size").get<int>() == 4);
    CHECK(agg.at("per_request").size() == reqs.size());
}

int main(int argc, char** argv) {
    g_golden = argc > 1 ? argv[1] : "tests/golden";
    for (auto& [name, fn] : registry()) {
        const int before = g_fail;
        fn();
        std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name.c_str());
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
