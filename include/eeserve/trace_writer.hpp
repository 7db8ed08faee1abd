// trace_writer.hpp — GPU-produced token records in the reference's workload
// trace format (one JSON object per request per line; the reference's
// trace_request_to_json / token_record_to_json, trace.hpp:99-121), so the
// unmodified reference simulate() can replay what the GPU decoded.
#pragma once

#include <cstdint>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "eeserve/errors.hpp"
#include "eeserve/trace.hpp"

namespace eeserve {

struct RecordedRequest {
    std::int64_t request_id = 0;
    double arrival_time_s = 0.0;
    int prompt_len = 0;
    std::vector<std::map<std::string, ModelTokenRecord>> tokens;  // per token: model -> record
};

// Doubles are written with 17 significant digits (exact round trip).
inline void write_trace_jsonl(const std::string& path, const std::vector<RecordedRequest>& reqs) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw ValidationError("cannot open workload file '" + path + "' for writing");
    for (const RecordedRequest& r : reqs) {
        std::fprintf(f, "{\"request_id\":%lld,\"arrival_time_s\":%.17g,\"prompt_len\":%d,\"tokens\":[",
                     (long long)r.request_id, r.arrival_time_s, r.prompt_len);
        for (size_t t = 0; t < r.tokens.size(); ++t) {
            std::fprintf(f, "%s{\"per_model\":{", t ? "," : "");
            bool first = true;
            for (const auto& [model, rec] : r.tokens[t]) {
                std::fprintf(f, "%s\"%s\":{\"final_token_id\":%d,\"observations\":[", first ? "" : ",", model.c_str(),
                             rec.final_token_id);
                first = false;
                for (size_t k = 0; k < rec.observations.size(); ++k) {
                    const ExitObservation& o = rec.observations[k];
                    std::fprintf(f, "%s{\"layer\":%d,\"token_id\":%d,\"confidence\":%.17g,\"logprob\":%.17g}",
                                 k ? "," : "", o.layer, o.token_id, o.confidence, o.logprob);
                }
                std::fprintf(f, "]}");
            }
            std::fprintf(f, "}}");
        }
        std::fprintf(f, "]}\n");
    }
    if (std::fclose(f) != 0) throw ValidationError("failed while writing workload file '" + path + "'");
}

}  // namespace eeserve
