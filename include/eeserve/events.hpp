// eeserve/events.hpp — the serving event log in the reference wire format.
//
// One JSON object per line with "t_s", "kind" and the kind's flat payload,
// exactly the schema of the reference's events.hpp
// (/root/reference/proj/include/eeserve/events.hpp:54-63):
//   request_start   {request_id}
//   prefill         {request_id, model, depth, duration_s}
//   token_emitted   {request_id, model, exit_layer, breached, unchanged, duration_s, logprob, energy_mwh}
//   weights_load    {model, from_depth, to_depth, bytes, duration_s, reason, loaded_bytes_after, energy_mwh}
//   model_switch    {from, to, reason}
//   eval_phase_*    {model}
//   reassess_*      {cycle}
//   request_complete{request_id, ttft_s, tpot_mean_s, latency_s, tokens}
// so the reference's aggregate() (metrics.hpp:51-145) rebuilds the engine's
// report from a GPU run's log: the tokens of one batched decode step share one
// t_s and count as one step of the step's width (metrics.hpp:85-93).
//
// Doubles are written with 17 significant digits (exact round trip); no JSON
// library is needed on the serving path.
#pragma once

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "eeserve/errors.hpp"

namespace eeserve {

class JsonFields {  // a flat JSON object under construction
public:
    JsonFields& num(const char* k, double v) {
        char b[40];
        std::snprintf(b, sizeof b, "%.17g", v);
        return raw(k, b);
    }
    JsonFields& i64(const char* k, std::int64_t v) { return raw(k, std::to_string(v)); }
    JsonFields& boolean(const char* k, bool v) { return raw(k, v ? "true" : "false"); }
    JsonFields& str(const char* k, const std::string& v) {
        std::string q = "\"";
        for (char c : v) {
            if (c == '"' || c == '\\') q += '\\';
            if ((unsigned char)c < 0x20) {
                char b[8];
                std::snprintf(b, sizeof b, "\\u%04x", (unsigned)(unsigned char)c);
                q += b;
                continue;
            }
            q += c;
        }
        return raw(k, q + "\"");
    }
    const std::string& body() const { return s_; }

private:
    JsonFields& raw(const char* k, const std::string& v) {
        if (!s_.empty()) s_ += ',';
        s_ += '"';
        s_ += k;
        s_ += "\":";
        s_ += v;
        return *this;
    }
    std::string s_;
};

struct EngineEvent {
    double t_s = 0.0;
    std::string kind;
    std::string fields;  // JsonFields::body()
};

inline std::string event_line(const EngineEvent& e) {
    JsonFields head;
    head.num("t_s", e.t_s).str("kind", e.kind);
    return "{" + (e.fields.empty() ? head.body() : e.fields + "," + head.body()) + "}";
}

inline void write_event_log(const std::vector<EngineEvent>& events, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw ValidationError("cannot open event log '" + path + "' for writing");
    for (const EngineEvent& e : events) out << event_line(e) << '\n';
    if (!out) throw ValidationError("failed while writing event log '" + path + "'");
}

}  // namespace eeserve
