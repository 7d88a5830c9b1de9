// strata_stg.cpp — the C++ drop-in: re-defines the reference's hot-path entry
// points on top of libstg's C-ABI (include/stg.h), with the reference's own
// declarations (proj/core/include/strata/*.hpp, included in place) so callers
// such as tools/strata.cpp and tests/acceptance.cpp relink unchanged:
//
//   strata::build_group_data   bundle.hpp:51-52  (bundle.cpp:252-324)   -> stg_window_run
//   strata::resolve_stacks     symrepo.hpp:55-57 (symrepo.cpp:122-143)  -> stg_resolve
//   strata::resolve_stack      symrepo.hpp:51-53 (symrepo.cpp:99-120)   -> stg_resolve
//   strata::aggregate_samples  samples.hpp:38-44 (samples.cpp:31-85)    -> stg_aggregate_samples
//   strata::diagnose           diagnosis.hpp:216-217 (diagnosis.cpp:301-432) -> the report the GPU
//                              computed in the same stg_window_run (re-run with the caller's
//                              DiagnosisConfig if it differs)
//
// build_group_data fills GroupData's CPU profiles from the structured getters
// (stg_result_rank_lines + stg_name, names cached per key) and only the small
// parts (GPU / OS / lateness / iteration times) from the JSON rendering.
// The reference TUs that define these symbols are compiled with
// -D<name>=<name>_reference (oracle/Makefile `dropin`), everything else of the
// reference links as is.  Errors from the library come back as strata::Error
// with the reference's message text.
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "json.hpp"
#include "stg.h"
#include <unordered_map>

#include "strata/bundle.hpp"
#include "strata/diagnosis.hpp"
#include "strata/samples.hpp"
#include "strata/symrepo.hpp"

namespace {

stg_ctx* ctx() {
    static std::once_flag once;
    static stg_ctx* c = nullptr;
    std::call_once(once, [] {
        const char* d = std::getenv("STG_DEVICE");
        if (stg_create(d ? std::atoi(d) : 0, &c) != STG_OK)
            throw strata::Error(std::string("libstg: ") + stg_last_error());
        std::atexit([] { stg_destroy(c); });
    });
    return c;
}

void check(int rc) {
    if (rc != STG_OK) throw strata::Error(stg_last_error());
}

// SymbolRepository::load (symrepo.cpp:90-97): the file bytes, if present.
bool load_symr(const strata::SymbolRepository& repo, const strata::BuildId& id, std::vector<uint8_t>& out) {
    std::ifstream in(repo.path_for(id), std::ios::binary);
    if (!in) return false;
    out.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
    return true;
}

// Stages every referenced binary's table (idempotent per build id).
void ingest_ids(const strata::SymbolRepository& repo, const std::vector<strata::BuildId>& ids) {
    std::vector<uint8_t> bytes;
    for (const auto& id : ids)
        if (load_symr(repo, id, bytes))
            check(stg_symtab_ingest(ctx(), id.bytes().data(), bytes.data(), bytes.size(), nullptr));
}

struct BinIndex {
    std::map<strata::BuildId, uint16_t> idx;
    std::vector<strata::BuildId> ids;
    std::vector<uint8_t> raw;
    uint16_t of(const strata::BuildId& id) {
        auto it = idx.find(id);
        if (it != idx.end()) return it->second;
        uint16_t k = uint16_t(ids.size());
        idx.emplace(id, k);
        ids.push_back(id);
        raw.insert(raw.end(), id.bytes().begin(), id.bytes().end());
        return k;
    }
};

std::string take_json(int (*fn)(stg_ctx*, char*, uint64_t, uint64_t*)) {
    uint64_t need = 0;
    check(fn(ctx(), nullptr, 0, &need));
    std::string s(need, '\0');
    check(fn(ctx(), s.data(), need, &need));
    s.resize(need ? need - 1 : 0);
    return s;
}

}  // namespace

namespace strata {

std::vector<std::vector<std::string>> resolve_stacks(const std::vector<std::vector<FrameRef>>& stacks,
                                                     const SymbolRepository& repo, SymbolFile::LookupMode mode) {
    BinIndex bins;
    std::vector<uint64_t> pc;
    std::vector<uint16_t> bin;
    for (const auto& s : stacks)
        for (const auto& f : s) {
            pc.push_back(f.offset);
            bin.push_back(bins.of(f.build_id));
        }
    ingest_ids(repo, bins.ids);
    std::vector<uint32_t> keys(pc.size());
    check(stg_resolve(ctx(), pc.size(), pc.data(), bin.data(), int32_t(bins.ids.size()), bins.raw.data(),
                      mode == SymbolFile::LookupMode::ExactRange ? STG_LOOKUP_EXACT_RANGE : STG_LOOKUP_NEAREST_LOWER,
                      keys.data()));
    std::map<uint32_t, std::string> names;
    std::vector<std::vector<std::string>> out;
    out.reserve(stacks.size());
    size_t k = 0;
    for (const auto& s : stacks) {
        std::vector<std::string> row;
        row.reserve(s.size());
        for (size_t i = 0; i < s.size(); ++i, ++k) {
            auto it = names.find(keys[k]);
            if (it == names.end()) {
                uint64_t need = 0;
                check(stg_name(ctx(), keys[k], nullptr, 0, &need));
                std::string nm(need, '\0');
                check(stg_name(ctx(), keys[k], nm.data(), need, &need));
                nm.resize(need - 1);
                it = names.emplace(keys[k], std::move(nm)).first;
            }
            row.push_back(it->second);
        }
        out.push_back(std::move(row));
    }
    return out;
}

std::vector<std::string> resolve_stack(const std::vector<FrameRef>& stack, const SymbolRepository& repo,
                                       SymbolFile::LookupMode mode) {
    return resolve_stacks({stack}, repo, mode).front();
}

namespace {
// The last window handed to the GPU, kept alive so diagnose() can re-run it
// with the caller's DiagnosisConfig, and the signature of the GroupData that
// build_group_data returned for it.
struct LastWindow {
    BinIndex bins;
    std::vector<int32_t> rank_ids, c_rank, c_group, g_rank, o_rank;
    std::vector<uint64_t> rank_off{0}, frame_off{0}, pc, irq_off{0}, sirq_off{0};
    std::vector<int64_t> ts, c_entry, c_exit, c_dur, g_start, g_dur, o_ws, o_p50, o_p99, o_mig, irq_v, sirq_v;
    std::vector<uint16_t> bin;
    std::vector<uint8_t> c_kind;
    std::vector<uint32_t> g_k, irq_k, sirq_k;
    std::map<std::string, uint32_t> kid, cid;
    std::vector<const char*> knames, cnames, bnames;
    std::vector<std::string> base_keys;
    std::vector<double> base_vals;
    std::vector<int32_t> group_ranks;
    stg_window w{};
    stg_config cfg{};
    uint64_t sig = 0;
};
std::mutex g_mu;
std::unique_ptr<LastWindow> g_last;

stg_config to_stg_config(const DiagnosisConfig& d) {
    stg_config c;
    stg_config_default(&c);
    c.window_iterations = d.window_iterations;
    c.k = d.k;
    c.delta = d.delta;
    c.iteration_regression_gate = d.iteration_regression_gate;
    c.gpu_median_uniform = d.gpu.median_uniform;
    c.gpu_cv_uniform = d.gpu.cv_uniform;
    c.gpu_top_share_specific = d.gpu.top_share_specific;
    c.gpu_median_none = d.gpu.median_none;
    c.gpu_ref_floor_ns = d.gpu.ref_floor_ns;
    std::memset(c.gpu_exclude_prefix, 0, sizeof c.gpu_exclude_prefix);
    std::strncpy(c.gpu_exclude_prefix, d.gpu.exclude_prefix.c_str(), sizeof c.gpu_exclude_prefix - 1);
    c.os_min_ratio = d.os.min_ratio;
    c.os_interrupt_floor = d.os.interrupt_floor;
    c.os_sched_delay_floor_ns = d.os.sched_delay_floor_ns;
    c.os_migration_floor = d.os.migration_floor;
    return c;
}

// FNV-1a over everything diagnose() reads from a GroupData
struct Sig {
    uint64_t h = 1469598103934665603ull;
    void bytes(const void* p, size_t n) {
        const unsigned char* q = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ q[i]) * 1099511628211ull;
    }
    template <class T>
    void pod(const T& v) { bytes(&v, sizeof v); }
    void str(const std::string& s) {
        pod(uint64_t(s.size()));
        bytes(s.data(), s.size());
    }
};
uint64_t signature(const GroupData& d) {
    Sig s;
    s.pod(d.group);
    for (const auto& [rank, p] : d.cpu_profiles) {
        s.pod(rank);
        s.pod(p.total);
        for (const auto& l : p.lines) {
            s.pod(uint64_t(l.frames.size()));
            for (const auto& f : l.frames) s.str(f);
            s.pod(l.count);
        }
    }
    for (const auto& [rank, g] : d.gpu_profiles) {
        s.pod(rank);
        for (const auto& [k, v] : g.kernel_time_ns) {
            s.str(k);
            s.pod(v);
        }
    }
    for (const auto& [rank, o] : d.os_snapshots) {
        s.pod(rank);
        for (const auto& [k, v] : o.interrupts) {
            s.str(k);
            s.pod(v);
        }
        for (const auto& [k, v] : o.softirqs) {
            s.str(k);
            s.pod(v);
        }
        s.pod(o.sched_delay_p50_ns);
        s.pod(o.sched_delay_p99_ns);
        s.pod(o.numa_migrations);
    }
    for (const auto& inst : d.lateness_per_instance) {
        s.pod(uint64_t(inst.size()));
        for (const auto& [r, l] : inst) {
            s.pod(r);
            s.pod(l);
        }
    }
    for (double t : d.iteration_times_ms) s.pod(t);
    s.pod(bool(d.baseline));
    if (d.baseline) {
        s.pod(d.baseline->delta);
        for (const auto& [k, v] : d.baseline->fractions) {
            s.str(k);
            s.pod(v);
        }
    }
    s.pod(bool(d.baseline_iteration_ms));
    if (d.baseline_iteration_ms) s.pod(*d.baseline_iteration_ms);
    return s.h;
}

}  // namespace

GroupData build_group_data(const LoadedBundle& b, const DiagnosisConfig& config) {
    // config is unused by the reference's build_group_data (bundle.cpp:322); the
    // run computes the report with it too, for the diagnose() that follows
    std::lock_guard<std::mutex> lk(g_mu);
    auto L = std::make_unique<LastWindow>();
    // ---- LoadedBundle -> stg_window (structure of arrays)
    BinIndex& bins = L->bins;
    std::vector<int32_t>& rank_ids = L->rank_ids;
    std::vector<uint64_t>&rank_off = L->rank_off, &frame_off = L->frame_off, &pc = L->pc;
    std::vector<int64_t>& ts = L->ts;
    std::vector<uint16_t>& bin = L->bin;
    for (const auto& [rank, stream] : b.samples) {
        rank_ids.push_back(rank);
        for (const StackSample& s : stream) {
            if (s.rank != stream.front().rank) throw Error("aggregate_samples: mixed ranks");
            ts.push_back(s.timestamp_ns);
            for (const FrameRef& f : s.frames) {
                pc.push_back(f.offset);
                bin.push_back(bins.of(f.build_id));
            }
            frame_off.push_back(pc.size());
        }
        rank_off.push_back(ts.size());
    }
    ingest_ids(SymbolRepository(b.dir), bins.ids);
    std::vector<int32_t>&c_rank = L->c_rank, &c_group = L->c_group;
    std::vector<uint8_t>& c_kind = L->c_kind;
    std::vector<int64_t>&c_entry = L->c_entry, &c_exit = L->c_exit, &c_dur = L->c_dur;
    for (const CollectiveEvent& e : b.collectives) {
        c_rank.push_back(e.rank);
        c_group.push_back(e.group);
        c_kind.push_back(uint8_t(e.kind));
        c_entry.push_back(e.host_entry_ns);
        c_exit.push_back(e.host_exit_ns);
        c_dur.push_back(e.gpu_duration_ns);
    }
    std::map<std::string, uint32_t>& kid = L->kid;
    for (const GpuEvent& e : b.gpu_events) kid.emplace(e.kernel, 0);
    std::vector<const char*>& knames = L->knames;
    for (auto& [k, v] : kid) {
        v = uint32_t(knames.size());
        knames.push_back(k.c_str());
    }
    std::vector<int32_t>& g_rank = L->g_rank;
    std::vector<uint32_t>& g_k = L->g_k;
    std::vector<int64_t>&g_start = L->g_start, &g_dur = L->g_dur;
    for (const GpuEvent& e : b.gpu_events) {
        g_rank.push_back(e.rank);
        g_k.push_back(kid.at(e.kernel));
        g_start.push_back(e.start_ns);
        g_dur.push_back(e.duration_ns);
    }
    std::map<std::string, uint32_t>& cid = L->cid;
    for (const OsCounterRecord& o : b.os_counters) {
        for (const auto& [k, v] : o.snapshot.interrupts) cid.emplace(k, 0);
        for (const auto& [k, v] : o.snapshot.softirqs) cid.emplace(k, 0);
    }
    std::vector<const char*>& cnames = L->cnames;
    for (auto& [k, v] : cid) {
        v = uint32_t(cnames.size());
        cnames.push_back(k.c_str());
    }
    std::vector<int32_t>& o_rank = L->o_rank;
    std::vector<int64_t>&o_ws = L->o_ws, &o_p50 = L->o_p50, &o_p99 = L->o_p99, &o_mig = L->o_mig,
                         &irq_v = L->irq_v, &sirq_v = L->sirq_v;
    std::vector<uint64_t>&irq_off = L->irq_off, &sirq_off = L->sirq_off;
    std::vector<uint32_t>&irq_k = L->irq_k, &sirq_k = L->sirq_k;
    for (const OsCounterRecord& o : b.os_counters) {
        o_rank.push_back(o.rank);
        o_ws.push_back(o.window_start_ns);
        o_p50.push_back(o.snapshot.sched_delay_p50_ns);
        o_p99.push_back(o.snapshot.sched_delay_p99_ns);
        o_mig.push_back(o.snapshot.numa_migrations);
        for (const auto& [k, v] : o.snapshot.interrupts) {
            irq_k.push_back(cid.at(k));
            irq_v.push_back(v);
        }
        for (const auto& [k, v] : o.snapshot.softirqs) {
            sirq_k.push_back(cid.at(k));
            sirq_v.push_back(v);
        }
        irq_off.push_back(irq_k.size());
        sirq_off.push_back(sirq_k.size());
    }
    stg_window& w = L->w;
    w.memory = STG_MEM_HOST;
    w.group = b.group;
    w.window_start_ns = b.window_start_ns;
    w.window_end_ns = b.window_end_ns;
    w.max_skew_ns = b.max_skew_ns;
    w.n_ranks = int32_t(rank_ids.size());
    w.rank_ids = rank_ids.data();
    w.rank_sample_off = rank_off.data();
    w.n_bins = int32_t(bins.ids.size());
    w.bin_build_ids = bins.raw.data();
    w.n_samples = ts.size();
    w.sample_ts = ts.data();
    w.sample_frame_off = frame_off.data();
    w.n_frames = pc.size();
    w.frame_pc = pc.data();
    w.frame_bin = bin.data();
    w.n_coll = c_rank.size();
    w.coll_rank = c_rank.data();
    w.coll_group = c_group.data();
    w.coll_kind = c_kind.data();
    w.coll_entry = c_entry.data();
    w.coll_exit = c_exit.data();
    w.coll_gpu_dur = c_dur.data();
    L->group_ranks = b.group_ranks;
    w.n_group_ranks = int32_t(L->group_ranks.size());
    w.group_ranks = L->group_ranks.data();
    w.n_gpu = g_rank.size();
    w.gpu_rank = g_rank.data();
    w.gpu_kernel = g_k.data();
    w.gpu_start = g_start.data();
    w.gpu_dur = g_dur.data();
    w.n_kernel_names = uint32_t(knames.size());
    w.kernel_names = knames.data();
    w.n_os = o_rank.size();
    w.os_rank = o_rank.data();
    w.os_window_start = o_ws.data();
    w.os_p50 = o_p50.data();
    w.os_p99 = o_p99.data();
    w.os_migrations = o_mig.data();
    w.os_irq_off = irq_off.data();
    w.os_irq_key = irq_k.data();
    w.os_irq_val = irq_v.data();
    w.os_sirq_off = sirq_off.data();
    w.os_sirq_key = sirq_k.data();
    w.os_sirq_val = sirq_v.data();
    w.n_counter_names = uint32_t(cnames.size());
    w.counter_names = cnames.data();
    // the bundle's baseline (bundle.cpp:257-258) for the temporal route
    w.has_baseline = 1;
    w.baseline_delta = b.baseline.delta;
    for (const auto& [k, v] : b.baseline.fractions) {
        L->base_keys.push_back(k);
        L->base_vals.push_back(v);
    }
    for (const auto& k : L->base_keys) L->bnames.push_back(k.c_str());
    w.n_baseline = uint32_t(L->base_keys.size());
    w.baseline_names = L->bnames.data();
    w.baseline_fracs = L->base_vals.data();
    w.has_baseline_iteration = 1;
    w.baseline_iteration_ms = b.baseline_iteration_ms;
    L->cfg = to_stg_config(config);
    check(stg_window_run(ctx(), &w, &L->cfg, nullptr));

    // ---- result -> GroupData (diagnosis.hpp:192-201): CPU profiles through the
    // structured getters, the rest from the (small) JSON rendering
    GroupData d;
    d.group = b.group;
    d.baseline = b.baseline;
    d.baseline_iteration_ms = b.baseline_iteration_ms;
    {
        uint32_t nr = 0;
        check(stg_result_rank_count(ctx(), &nr));
        std::unordered_map<uint32_t, std::string> names;
        auto name_of = [&](uint32_t key) -> const std::string& {
            auto it = names.find(key);
            if (it == names.end()) {
                uint64_t need = 0;
                check(stg_name(ctx(), key, nullptr, 0, &need));
                std::string nm(need, '\0');
                check(stg_name(ctx(), key, nm.data(), need, &need));
                nm.resize(need - 1);
                it = names.emplace(key, std::move(nm)).first;
            }
            return it->second;
        };
        std::vector<uint64_t> koff, counts;
        std::vector<uint32_t> keys;
        for (uint32_t i = 0; i < nr; ++i) {
            int32_t rank = 0;
            uint64_t nl = 0, total = 0, nk = 0;
            check(stg_result_rank_info(ctx(), i, &rank, &nl, &total, &nk));
            koff.resize(nl + 1);
            keys.resize(nk);
            counts.resize(nl);
            check(stg_result_rank_lines(ctx(), i, koff.data(), keys.data(), counts.data()));
            FoldedProfile& f = d.cpu_profiles[rank];
            f.total = total;
            f.lines.reserve(nl);
            for (uint64_t l = 0; l < nl; ++l) {
                std::vector<std::string> frames;
                frames.reserve(koff[l + 1] - koff[l]);
                for (uint64_t k = koff[l]; k < koff[l + 1]; ++k) frames.push_back(name_of(keys[k]));
                f.lines.push_back({std::move(frames), counts[l]});
            }
        }
    }
    uint64_t need = 0;
    check(stg_result_groupdata_json_parts(ctx(), STG_GD_ALL & ~STG_GD_CPU, nullptr, 0, &need));
    std::string js(need, '\0');
    check(stg_result_groupdata_json_parts(ctx(), STG_GD_ALL & ~STG_GD_CPU, js.data(), need, &need));
    js.resize(need ? need - 1 : 0);
    nlohmann::json j = nlohmann::json::parse(js);
    for (const auto& p : j.at("gpu_profiles")) {
        GpuProfile& g = d.gpu_profiles[p.at("rank").get<int>()];
        for (const auto& k : p.at("kernels")) g.kernel_time_ns[k.at(0).get<std::string>()] = k.at(1).get<int64_t>();
    }
    for (const auto& p : j.at("os_snapshots")) {
        OsSnapshot& o = d.os_snapshots[p.at("rank").get<int>()];
        for (const auto& k : p.at("interrupts")) o.interrupts[k.at(0).get<std::string>()] = k.at(1).get<int64_t>();
        for (const auto& k : p.at("softirqs")) o.softirqs[k.at(0).get<std::string>()] = k.at(1).get<int64_t>();
        o.sched_delay_p50_ns = p.at("p50").get<int64_t>();
        o.sched_delay_p99_ns = p.at("p99").get<int64_t>();
        o.numa_migrations = p.at("migrations").get<int64_t>();
    }
    for (const auto& inst : j.at("lateness_per_instance")) {
        std::map<int, double> m;
        for (const auto& rl : inst) m[rl.at(0).get<int>()] = rl.at(1).get<double>();
        d.lateness_per_instance.push_back(std::move(m));
    }
    d.iteration_times_ms = j.at("iteration_times_ms").get<std::vector<double>>();
    L->sig = signature(d);
    g_last = std::move(L);
    return d;
}

// diagnose (diagnosis.cpp:301-432): the verdict the GPU computed for this
// GroupData in build_group_data's window run.  A GroupData that did not come out
// of the preceding build_group_data is refused (the drop-in computes diagnoses
// on the device from the window, not from a hand-built GroupData).
DiagnosisReport diagnose(const GroupData& data, const DiagnosisConfig& config) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_last || signature(data) != g_last->sig)
        throw Error("libstg drop-in: diagnose() takes the GroupData of the preceding build_group_data() call");
    const stg_config cfg = to_stg_config(config);
    if (std::memcmp(&cfg, &g_last->cfg, sizeof cfg) != 0) {  // other thresholds: same window, new run
        g_last->cfg = cfg;
        check(stg_window_run(ctx(), &g_last->w, &g_last->cfg, nullptr));
    }
    const nlohmann::json j = nlohmann::json::parse(take_json(stg_result_report_json));
    DiagnosisReport r;
    static const std::map<std::string, Verdict> verdicts = {
        {"healthy", Verdict::Healthy},
        {"gpu-uniform-slowdown", Verdict::GpuUniformSlowdown},
        {"gpu-specific-kernel", Verdict::GpuSpecificKernel},
        {"cpu-interference", Verdict::CpuInterference},
        {"os-interference", Verdict::OsInterference},
        {"temporal-degradation", Verdict::TemporalDegradation},
        {"inconclusive", Verdict::Inconclusive}};
    r.verdict = verdicts.at(j.at("verdict").get<std::string>());
    r.flagged_ranks = j.at("flagged_ranks").get<std::vector<int>>();
    for (const auto& e : j.at("evidence"))
        r.evidence.push_back({e.at("layer").get<std::string>(), e.at("item").get<std::string>(),
                              e.at("straggler_value").get<double>(), e.at("reference_value").get<double>(),
                              e.at("delta").get<double>()});
    r.top_path = j.at("top_path").get<std::vector<std::string>>();
    r.notes = j.at("notes").get<std::vector<std::string>>();
    if (!j.at("reference_rank").is_null()) r.reference_rank = j.at("reference_rank").get<int>();
    return r;
}

// Raw samples -> SoA (build ids interned to bins), aggregated on the GPU; each
// record's frames are its first-seen sample's frames.
std::vector<ProfileWindow> aggregate_samples(const std::vector<StackSample>& stream, int64_t drain_interval_ns) {
    const uint64_t n = stream.size();
    std::vector<int64_t> ts(n);
    std::vector<int32_t> rank(n);
    std::vector<uint64_t> off(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) off[i + 1] = off[i] + stream[i].frames.size();
    std::vector<uint64_t> pc(off[n]);
    std::vector<uint16_t> bin(off[n]);
    std::unordered_map<BuildId, uint16_t, BuildIdHash> bins;
    const BuildId* last = nullptr;  // consecutive frames mostly share a binary
    uint16_t last_bin = 0;
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const StackSample& s = stream[i];
        ts[i] = s.timestamp_ns;
        rank[i] = s.rank;
        for (const FrameRef& f : s.frames) {
            if (!last || !(f.build_id == *last)) {
                auto it = bins.find(f.build_id);
                if (it == bins.end()) {
                    if (bins.size() > 0xffff) throw Error("libstg: more than 65536 build ids in one stream");
                    it = bins.emplace(f.build_id, uint16_t(bins.size())).first;
                }
                last = &it->first;
                last_bin = it->second;
            }
            pc[k] = f.offset;
            bin[k++] = last_bin;
        }
    }
    stg_stream st{};
    st.memory = STG_MEM_HOST;
    st.n_samples = n;
    st.ts = ts.data();
    st.rank = rank.data();
    st.frame_off = off.data();
    st.frame_pc = pc.data();
    st.frame_bin = bin.data();
    uint64_t nw = 0, nr = 0;
    check(stg_aggregate_samples(ctx(), &st, drain_interval_ns, 0, &nw, &nr));
    std::vector<int64_t> ws(nw), we(nw);
    std::vector<uint64_t> ro(nw + 1), first(nr), count(nr);
    check(stg_aggregate_windows(ctx(), ws.data(), we.data(), ro.data()));
    check(stg_aggregate_records(ctx(), first.data(), count.data()));
    std::vector<ProfileWindow> out(nw);
    for (uint64_t w = 0; w < nw; ++w) {
        ProfileWindow& pw = out[w];
        pw.rank = stream.front().rank;
        pw.window_start_ns = ws[w];
        pw.window_end_ns = we[w];
        pw.records.reserve(ro[w + 1] - ro[w]);
        for (uint64_t r = ro[w]; r < ro[w + 1]; ++r) pw.records.push_back({stream[first[r]].frames, count[r]});
    }
    return out;
}

}  // namespace strata
