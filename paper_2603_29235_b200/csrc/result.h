// result.h — host-side view of one window's result (GroupData + report).
#pragma once

#include <algorithm>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "stg_internal.h"

namespace stg {

struct Evidence {
    std::string layer, item;
    double straggler_value = 0, reference_value = 0, delta = 0;
};

struct Report {
    int verdict = STG_VERDICT_HEALTHY;
    std::vector<int> flagged_ranks;
    std::vector<Evidence> evidence;
    std::vector<std::string> top_path;
    std::optional<int> reference_rank;
    std::vector<std::string> notes;
};

struct OsAcc {
    std::map<std::string, int64_t> interrupts, softirqs;
    int64_t p50 = 0, p99 = 0, migrations = 0;
};

// Everything a window run leaves behind.  Bulk arrays stay on the device
// (ctx buffers); what the decision ladder and the getters need is mirrored here.
struct Result {
    int group = 0;
    int32_t rank_span = 0;  // dense rank index space [0, rank_span)
    // ---- collectives
    bool have_offsets = false;
    std::vector<int64_t> offsets;   // [rank_span]
    std::vector<uint8_t> has_offset;
    uint64_t n_instances = 0, n_windowed = 0;
    std::vector<double> iteration_times_ms;
    // straggler stats per rank (dense)
    std::vector<uint8_t> lat_present;     // rank appears in some windowed instance
    std::vector<double> mean_lat_all;     // over all instances containing it (median_lateness_rank)
    std::vector<double> mean_lat_alert;   // over instances with >= 2 ranks (StragglerAlert)
    std::vector<double> z_mean;
    std::vector<uint64_t> flag_count;
    std::vector<uint8_t> has_z;
    // ---- gpu / os
    std::map<int, std::map<std::string, int64_t>> gpu;
    std::map<int, OsAcc> os;
    // ---- cpu profiles
    std::vector<int32_t> cpu_rank_ids;  // ranks with a profile (ascending)
    std::vector<uint32_t> cpu_rank_index;  // index into window ranks
    std::vector<uint64_t> cpu_totals;
    uint64_t n_lines = 0, n_seq = 0, n_names = 0, n_unknown = 0, f_used = 0, n_gid = 0;
    uint32_t n_window_ranks = 0;
    int agg_attempts = 0;
    uint64_t pfx_hits = 0, pfx_misses = 0;
    uint32_t verified = 0, verify_retries = 0;
    uint64_t f_nd_bound = 1;  // bound on the (sequence, distinct name) pairs of the fold
    // host mirror of the folded lines, downloaded once on first use (getters)
    struct HostFold {
        bool ok = false;
        std::vector<uint64_t> lkey, lcount, seq_off, line_off;
        std::vector<uint32_t> dense_rep, arena;
    } hf;
    std::string svg_text;  // last rendered flame graph (two-call size query)
    uint64_t svg_key = ~0ull;
    // name space: final rank -> string
    std::vector<uint64_t> unk_final;       // final rank of each distinct unknown label (sorted)
    std::vector<std::string> unk_labels;   // labels in the same order
    const Dict* dict = nullptr;
    std::string name_of(uint32_t final_rank) const;
    // ---- baseline
    bool has_baseline = false;
    double baseline_delta = 0.005;
    std::map<std::string, double> baseline;
    bool has_baseline_iteration = false;
    double baseline_iteration_ms = 0;
    // ---- report
    Report report;
    bool waterline_done = false;
    std::string waterline_json;
    uint64_t wl_flags = 0, wl_F = 0;
    // distributed waterline: global name space kept for lazy rendering
    bool wl_dist = false;
    uint64_t wl_NG = 0;
    std::vector<uint64_t> g_lab_final;
    std::vector<std::string> g_lab;
    uint64_t wl_NGF = 0;  // global name space; device byte map "wl_umap" marks the waterline's names
    std::string gname(uint32_t g) const {
        auto it = std::lower_bound(g_lab_final.begin(), g_lab_final.end(), uint64_t(g));
        if (it != g_lab_final.end() && *it == g) return g_lab[size_t(it - g_lab_final.begin())];
        return std::string((*dict)[g - uint64_t(it - g_lab_final.begin())]);
    }
    stg_run_stats stats{};
    // folded-text artifacts (stg_render.cu): last rendering kept on the device
    bool render_valid = false, render_unk_ready = false;
    int render_kind = -1;
    int32_t render_a = 0, render_b = 0;
    uint64_t render_len = 0;
};

// stg_report.cpp (nlohmann/json, like the reference's serialisers)
const char* verdict_name(int v);
std::string report_json_dump2(const Report& p);
std::string report_text(const Report& p);

}  // namespace stg
