// stg_report.cpp — DiagnosisReport renderings, byte-identical to the reference:
//   to_json  diagnosis.cpp:437-455  nlohmann::json object, dump(2)
//   to_text  diagnosis.cpp:457-481  std::ostream formatting (default precision)
// The reference serialises with nlohmann/json (3.11.3, its only third-party
// dependency); rendering with the same library makes the key
// order, indentation and shortest round-trip double formatting the same bytes.
#include <sstream>

#include "json.hpp"
#include "result.h"

namespace stg {

const char* verdict_name(int v) {
    static const char* names[] = {"healthy",          "gpu-uniform-slowdown", "gpu-specific-kernel",
                                  "cpu-interference", "os-interference",      "temporal-degradation",
                                  "inconclusive"};
    return v >= 0 && v < 7 ? names[v] : "unknown";
}

std::string report_json_dump2(const Report& p) {
    nlohmann::json ev = nlohmann::json::array();
    for (const auto& e : p.evidence)
        ev.push_back({{"layer", e.layer},
                      {"item", e.item},
                      {"straggler_value", e.straggler_value},
                      {"reference_value", e.reference_value},
                      {"delta", e.delta}});
    nlohmann::json j{{"verdict", verdict_name(p.verdict)},
                     {"flagged_ranks", p.flagged_ranks},
                     {"evidence", ev},
                     {"top_path", p.top_path},
                     {"notes", p.notes}};
    if (p.reference_rank)
        j["reference_rank"] = *p.reference_rank;
    else
        j["reference_rank"] = nullptr;
    return j.dump(2);
}

std::string report_text(const Report& p) {
    std::ostringstream os;
    os << "verdict: " << verdict_name(p.verdict) << "\n";
    os << "flagged ranks:";
    if (p.flagged_ranks.empty()) os << " none";
    for (int r : p.flagged_ranks) os << " " << r;
    os << "\n";
    if (p.reference_rank) os << "reference rank: " << *p.reference_rank << "\n";
    if (!p.top_path.empty()) {
        os << "top path: ";
        for (size_t i = 0; i < p.top_path.size(); ++i) {
            if (i) os << ";";
            os << p.top_path[i];
        }
        os << "\n";
    }
    if (!p.evidence.empty()) {
        os << "evidence (" << p.evidence.size() << " items):\n";
        for (const auto& e : p.evidence)
            os << "  [" << e.layer << "] " << e.item << ": " << e.straggler_value << " vs " << e.reference_value
               << " (delta " << e.delta << ")\n";
    }
    for (const auto& n : p.notes) os << "note: " << n << "\n";
    return os.str();
}

}  // namespace stg
