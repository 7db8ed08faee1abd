// GPU records through the reference: the decision layer pinned on real GPU output
// (SURVEY §4 implication 3).
//
//  1. Record: every request's prompt prefilled and its tokens decoded on the
//     B200 with every exit head evaluated (EEB_PROFILE, batch 1) for each
//     model of the repository, written as a reference-format workload trace
//     (eeserve/trace_writer.hpp; the reference's trace.hpp:99-121 schema).
//  2. Reference: the UNMODIFIED reference simulate() (oracle/_ref/libeeref.so)
//     replays that trace (helios / ee_single / vanilla modes).
//  3. Live: BatchedEngine (Simulator::run's control flow) over ProfileBackend —
//     the same requests decoded again on the GPU, the reference's token rule
//     applied to the live records (backend.hpp) — at batch 1.
//  The two reports must agree: exit tables, action counts (load-more / switch
//  / reassess), unchanged fraction, perplexity, throughput and TTFT (modelled
//  times on both sides), and the PHT histograms; and the live records must be
//  bit-identical to the recorded ones (the decode is deterministic and batch
//  invariant).
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>

#include <json.hpp>

#include "eeserve/engine.hpp"
#include "eeserve/trace_writer.hpp"

using namespace eeserve;
using Json = nlohmann::json;

extern "C" {
int ref_simulate(const char*, const char*, const char*, const char*, const char*, char*, int);
const char* ref_last_error();
}

static int g_checks = 0, g_fail = 0;
#define CHECK(c)                                                                    \
    do {                                                                            \
        ++g_checks;                                                                 \
        if (!(c)) {                                                                 \
            ++g_fail;                                                               \
            std::fprintf(stderr, "%s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
        }                                                                           \
    } while (0)

static bool approx(double a, double b, double rel) { return std::fabs(a - b) <= rel * std::max(1.0, std::fabs(b)); }

struct Shape {
    std::string id;
    int layers;
    std::vector<int> exits;
    int d, heads, ffn, vocab;
    std::uint64_t seed;
    double thr, t_layer;
};

static ModelSpec spec_of(const Shape& m) {
    ModelSpec s;
    s.id = m.id;
    s.num_layers = m.layers;
    s.exit_layers = m.exits;
    s.per_layer_weight_bytes = (4LL * m.d * m.d + 2LL * m.d * m.ffn) * 2 + 2LL * m.d * 4;
    s.base_weight_bytes = (std::int64_t)m.vocab * m.d * 2 * (1 + (std::int64_t)m.exits.size());
    s.kv_bytes_per_token_per_layer = 4LL * m.d;
    s.t_decode_per_layer_s = m.t_layer;
    s.t_prefill_per_layer_per_token_s = m.t_layer / 16.0;
    s.energy_per_layer_per_token_mwh = 0.5;
    s.repo_metrics["throughput"] = m.thr;
    s.arch.d_model = m.d;
    s.arch.n_heads = m.heads;
    s.arch.n_kv_heads = m.heads;
    s.arch.d_ffn = m.ffn;
    s.arch.vocab = m.vocab;
    s.arch.dtype = EEB_BF16;
    s.arch.seed = m.seed;
    validate_model_spec(s);
    return s;
}

static void write_repo_json(const ModelRepository& repo, const std::string& path) {
    Json models = Json::array();
    for (const auto& [id, s] : repo.models)
        models.push_back({{"id", id},
                          {"num_layers", s.num_layers},
                          {"exit_layers", s.exit_layers},
                          {"base_weight_bytes", s.base_weight_bytes},
                          {"per_layer_weight_bytes", s.per_layer_weight_bytes},
                          {"kv_bytes_per_token_per_layer", s.kv_bytes_per_token_per_layer},
                          {"t_decode_per_layer_s", s.t_decode_per_layer_s},
                          {"t_prefill_per_layer_per_token_s", s.t_prefill_per_layer_per_token_s},
                          {"energy_per_layer_per_token_mwh", s.energy_per_layer_per_token_mwh},
                          {"repo_metrics", {{"throughput", s.repo_metrics.at("throughput")}}}});
    std::ofstream(path) << Json{{"models", models}, {"metric_directions", {{"throughput", "higher_better"}}}}.dump(1);
}

int main() {
    const std::vector<Shape> shapes = {{"small", 6, {2, 4, 6}, 256, 4, 512, 512, 31, 2.0, 1e-4},
                                       {"large", 8, {4, 8}, 256, 4, 768, 512, 32, 1.0, 1.4e-4}};
    ModelRepository repo;
    for (const auto& m : shapes) repo.models[m.id] = spec_of(m);
    repo.metric_directions["throughput"] = MetricDirection::higher_better;
    const std::string repo_path = "/tmp/eeb_replay_repo.json", trace_path = "/tmp/eeb_replay_trace.jsonl";
    write_repo_json(repo, repo_path);
    const std::uint64_t token_seed = 20260819;
    const int S = 64;

    // ---- 1. record every (request, model) on the GPU ------------------------------
    std::vector<RequestSpec> reqs;
    for (int i = 0; i < 80; ++i) reqs.push_back({i, 6 + i % 4, 8 + i % 3});
    std::vector<RecordedRequest> trace;
    {
        CudaBackend gpu(0);
        for (const auto& [id, s] : repo.models) {
            gpu.register_model(s, 1, S);
            gpu.load(id, s.num_layers);
        }
        for (const auto& r : reqs) {
            RecordedRequest rr{r.request_id, 0.0, r.prompt_len, {}};
            rr.tokens.resize(r.num_tokens);
            for (const auto& [id, s] : repo.models) {
                PrefillRows pr;
                pr.slots = {0};
                std::vector<int32_t> p(r.prompt_len);
                for (int k = 0; k < r.prompt_len; ++k) p[k] = synthetic_token(token_seed, r.request_id, k, s.arch.vocab);
                pr.prompts.push_back(p);
                gpu.prefill(id, s.num_layers, pr);
                for (int t = 0; t < r.num_tokens; ++t) {
                    const int pos = r.prompt_len + t;
                    StepRows rows;
                    rows.slots = {0};
                    rows.tokens = {synthetic_token(token_seed, r.request_id, pos, s.arch.vocab)};
                    rows.positions = {pos};
                    rows.request_ids = {r.request_id};
                    rows.token_index = {t};
                    const StepOutcome o = gpu.step(id, 0, TokenPolicy::profile, 0.7, rows);
                    rr.tokens[t][id] = o.records.at(0);
                }
            }
            trace.push_back(std::move(rr));
        }
    }
    write_trace_jsonl(trace_path, trace);

    // ---- 2 + 3. reference simulate() over the trace vs the engine decoding live -----
    struct Case {
        const char* mode_str;
        Mode mode;
        const char* model;
    };
    const MemoryConfig mem{4'000'000'000, 100'000'000, S, 8.4e9};
    PolicyConfig pol;
    pol.k = 2;
    pol.n_eval_requests = 5;
    pol.ri = 30;
    pol.window = 20;
    pol.cbc_max = 5;
    const std::string pj = Json{{"k", pol.k}, {"n_eval_requests", pol.n_eval_requests}, {"ri", pol.ri},
                                {"window", pol.window}, {"cbc_max", pol.cbc_max}}.dump();
    const std::string mj = Json{{"capacity_bytes", mem.capacity_bytes}, {"reserve_bytes", mem.reserve_bytes},
                                {"max_seq_len", mem.max_seq_len}, {"bandwidth_bytes_per_s", mem.bandwidth_bytes_per_s}}
                               .dump();
    for (const Case& c : {Case{"helios", Mode::helios, ""}, Case{"ee_single:small", Mode::ee_single, "small"},
                          Case{"ee_single:large", Mode::ee_single, "large"}, Case{"vanilla:small", Mode::vanilla, "small"}}) {
        std::vector<char> buf(1 << 24);
        const int rc = ref_simulate(repo_path.c_str(), trace_path.c_str(), c.mode_str, pj.c_str(), mj.c_str(), buf.data(),
                                    (int)buf.size());
        CHECK(rc > 0);
        if (rc <= 0) {
            std::fprintf(stderr, "ref_simulate(%s): %s\n", c.mode_str, ref_last_error());
            continue;
        }
        const Json ref = Json::parse(buf.data());
        const Json& rr = ref.at("report");

        CudaBackend gpu(0);
        ProfileBackend be(gpu);
        std::int64_t mismatched = 0, seen = 0;
        be.recorder = [&](const std::string& model, std::int64_t rid, int t, const ModelTokenRecord& rec) {
            const ModelTokenRecord& want = trace.at((size_t)rid).tokens.at((size_t)t).at(model);
            ++seen;
            bool same = rec.final_token_id == want.final_token_id && rec.observations.size() == want.observations.size();
            for (size_t k = 0; same && k < rec.observations.size(); ++k) {
                const ExitObservation &a = rec.observations[k], &b = want.observations[k];
                same = a.layer == b.layer && a.token_id == b.token_id && a.confidence == b.confidence &&
                       a.logprob == b.logprob;
            }
            mismatched += same ? 0 : 1;
        };
        EngineConfig cfg;
        cfg.mem = mem;
        cfg.policy = pol;
        cfg.mode = ModeSpec{c.mode, c.model};
        cfg.max_batch = 1;
        cfg.max_seq_len = S;
        cfg.token_seed = token_seed;
        BatchedEngine eng(repo, be, cfg);
        const EngineReport rep = eng.run(reqs);

        CHECK(seen > 0 && mismatched == 0);  // live decode == recorded decode, bit for bit
        const Json& agg = rr.at("aggregates");
        CHECK(approx(rep.perplexity, agg.at("perplexity").get<double>(), 1e-12));
        CHECK(approx(rep.unchanged_fraction, agg.at("unchanged_fraction").get<double>(), 1e-12));
        CHECK(approx(rep.throughput_tok_s, agg.at("throughput_tok_s").get<double>(), 1e-9));
        CHECK(approx(rep.mean_ttft_s, agg.at("mean_ttft_s").get<double>(), 1e-9));
        CHECK(agg.at("achieved_batch_size").get<int>() == rep.achieved_batch_size);
        const Json& ac = rr.at("action_counts");
        const std::int64_t ref_ld = ac.at("ld").get<std::int64_t>(), ref_sw = ac.at("sw").get<std::int64_t>();
        CHECK(rep.ld_count == ref_ld);
        CHECK(rep.sw_count == ref_sw);
        int rows = 0;
        for (auto& [m, per] : rr.at("exit_table").items())
            for (auto& [layer, pct] : per.items()) {
                ++rows;
                const auto mi = rep.exit_table.find(m);
                CHECK(mi != rep.exit_table.end() && mi->second.count(std::stoi(layer)) &&
                      approx(mi->second.at(std::stoi(layer)), pct.get<double>(), 1e-12));
            }
        CHECK(rows > 0);
        for (auto& [m, e] : ref.at("pht").items()) {
            const auto it = rep.pht.entries.find(m);
            CHECK(it != rep.pht.entries.end());
            if (it == rep.pht.entries.end()) continue;
            CHECK(it->second.token_count == e.at("token_count").get<std::int64_t>());
            CHECK(approx(it->second.sum_neg_logprob, e.at("sum_neg_logprob").get<double>(), 1e-12));
            for (auto& [layer, cnt] : e.at("exit_hist").at("counts").items())
                CHECK(it->second.exit_hist.counts.count(std::stoi(layer)) &&
                      it->second.exit_hist.counts.at(std::stoi(layer)) == cnt.get<std::int64_t>());
        }
        std::printf("%-16s tokens %lld, ld %lld (ref %lld), sw %lld (ref %lld), perplexity %.6f, exit rows %d, "
                    "records %lld (%lld differ)\n",
                    c.mode_str, (long long)rep.tokens, (long long)rep.ld_count, (long long)ref_ld,
                    (long long)rep.sw_count, (long long)ref_sw, rep.perplexity, rows, (long long)seen,
                    (long long)mismatched);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
