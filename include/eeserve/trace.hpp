// eeserve/trace.hpp — per-token exit observations and the two exit rules.
//
// Interface of /root/reference/proj/include/eeserve/trace.hpp:17-97.  In the
// reference these records come from a pre-computed trace; here the GPU
// backend (eeserve/backend.hpp) produces them from real exit heads.
// JSONL trace I/O is outside the hot path (SURVEY §8f "next").
//
// PROVENANCE: a verbatim-semantics port of /root/reference/proj/include/eeserve/trace.hpp:17-97
// (same identifiers, control flow and error strings; JSON I/O dropped).  It is
// the reference host API that the drop-in keeps unchanged, not new work; its
// behaviour is pinned against the compiled reference (tests/cpp/test_host.cpp).
#pragma once

#include <cstdint>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "eeserve/model_spec.hpp"

namespace eeserve {

/// One exit head's verdict on one token (trace.hpp:17-22).
struct ExitObservation {
    int layer = 0;
    int token_id = 0;
    double confidence = 0.0;  // max softmax probability
    double logprob = 0.0;     // log-probability of token_id at this head
};

/// Every head of one model on one token, shallow to deep, plus the token the
/// full model settles on (trace.hpp:26-35).
struct ModelTokenRecord {
    int final_token_id = 0;
    std::vector<ExitObservation> observations;

    const ExitObservation& at_layer(int layer) const {
        for (const auto& o : observations)
            if (o.layer == layer) return o;
        throw DomainError("no observation at layer " + std::to_string(layer));
    }
};

struct TokenRecord {
    std::map<std::string, ModelTokenRecord> per_model;

    const ModelTokenRecord& for_model(const std::string& model_id) const {
        const auto it = per_model.find(model_id);
        if (it == per_model.end())
            throw DomainError("token record has no entry for model '" + model_id + "'");
        return it->second;
    }
};

struct TraceRequest {
    std::int64_t request_id = 0;
    double arrival_time_s = 0.0;
    int prompt_len = 0;
    std::vector<TokenRecord> tokens;
    int num_tokens() const { return static_cast<int>(tokens.size()); }
};

struct Trace {
    std::vector<TraceRequest> requests;
};

/// Position of `depth` in the exit ladder; DomainError when it is not an exit.
inline std::size_t exit_index(const std::vector<int>& exit_layers, int depth) {
    for (std::size_t i = 0; i < exit_layers.size(); ++i)
        if (exit_layers[i] == depth) return i;
    throw DomainError("depth " + std::to_string(depth) + " is not an exit layer");
}

/// Introspective rule: the shallowest head at or above the threshold (>=);
/// the final head is a forced exit (trace.hpp:69-76).
inline const ExitObservation& earliest_confident_obs(const ModelTokenRecord& rec, double threshold) {
    if (rec.observations.empty()) throw DomainError("token record has no observations");
    for (const auto& o : rec.observations)
        if (o.confidence >= threshold) return o;
    return rec.observations.back();
}

inline int earliest_confident_exit(const TokenRecord& rec, const std::string& model_id,
                                   double threshold) {
    return earliest_confident_obs(rec.for_model(model_id), threshold).layer;
}

/// Greedy (flat) rule: the head at exactly `depth`, else the deepest head
/// below it (trace.hpp:86-97; the reference also logs a warning).
inline const ExitObservation& observation_for_depth(const ModelTokenRecord& rec, int depth) {
    const ExitObservation* below = nullptr;
    for (const auto& o : rec.observations) {
        if (o.layer == depth) return o;
        if (o.layer < depth) below = &o;
    }
    if (!below) throw DomainError("no observation at or below layer " + std::to_string(depth));
    return *below;
}

}  // namespace eeserve
