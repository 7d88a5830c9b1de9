// ref_harness.cpp — TEST INFRASTRUCTURE ONLY (oracle side, never the product).
//
// A thin extern "C" driver around the UNMODIFIED reference ("strata",
// /root/reference/proj/core) compiled in place by oracle/Makefile into
// oracle/_ref/libstrata_ref.so.  It lets tests and bench.py's cpu_baseline /
// `--impl reference` leg feed the reference the very same structure-of-arrays
// window (include/stg.h) that the GPU library consumes:
//
//   ref_sim_*        simulate(default_spec(...)) (simulate.cpp:272-545) exported as
//                    an stg_window + SYMR payloads — the labeled fixture generator.
//   ref_window_run   stg_window -> LoadedBundle (bundle.hpp:23-42) -> build_group_data
//                    (bundle.cpp:252-324) -> diagnose (diagnosis.cpp:301-432), timed,
//                    rendered as canonical JSON (same layout as stg_result_*_json).
//   ref_* verbs      single reference functions for unit parity (lookup, fold, match…).
//
// Nothing here re-implements reference logic: every result comes from the
// reference's own functions.  The rank-parallel mode only runs the reference's
// reentrant per-rank calls (aggregate_samples + to_folded) on std::threads, as
// BASELINE.md §4(b) plans, and merges them exactly as build_group_data does.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <filesystem>
#include <map>
#include <random>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"
#include "stg.h"
#include "strata/bundle.hpp"
#include "strata/svg.hpp"
#include "strata/collective.hpp"
#include "strata/diagnosis.hpp"
#include "strata/folded.hpp"
#include "strata/samples.hpp"
#include "strata/scenario.hpp"
#include "strata/symfile.hpp"
#include "strata/symrepo.hpp"

using namespace strata;
using nlohmann::json;
namespace fs = std::filesystem;

namespace {

void set_err(char* err, int cap, const std::string& m) {
    if (err && cap > 0) {
        std::snprintf(err, size_t(cap), "%s", m.c_str());
    }
}

BuildId id_at(const uint8_t* p) {
    std::array<uint8_t, BuildId::kSize> a{};
    std::memcpy(a.data(), p, BuildId::kSize);
    return BuildId(a);
}

// ----------------------------------------------------------------- simulator
struct SimHandle {
    SimulationResult res;
    std::vector<std::vector<uint8_t>> symr;
    std::string labels;
    // SoA storage
    std::vector<int32_t> rank_ids;
    std::vector<uint64_t> rank_sample_off;
    std::vector<uint8_t> bin_ids;
    std::vector<int64_t> ts;
    std::vector<uint64_t> frame_off;
    std::vector<uint64_t> pc;
    std::vector<uint16_t> bin;
    std::vector<int32_t> c_rank, c_group;
    std::vector<uint8_t> c_kind;
    std::vector<int64_t> c_entry, c_exit, c_dur;
    std::vector<int32_t> group_ranks;
    std::vector<int32_t> g_rank;
    std::vector<uint32_t> g_kernel;
    std::vector<int64_t> g_start, g_dur;
    std::vector<std::string> kernel_names;
    std::vector<const char*> kernel_cstr;
    std::vector<int32_t> o_rank;
    std::vector<int64_t> o_ws, o_p50, o_p99, o_mig;
    std::vector<uint64_t> o_irq_off, o_sirq_off;
    std::vector<uint32_t> o_irq_key, o_sirq_key;
    std::vector<int64_t> o_irq_val, o_sirq_val;
    std::vector<std::string> counter_names;
    std::vector<const char*> counter_cstr;
    std::vector<std::string> base_names;
    std::vector<const char*> base_cstr;
    std::vector<double> base_fracs;
    stg_window win{};
};

void build_soa(SimHandle& h) {
    const SimulationResult& r = h.res;
    std::map<BuildId, uint16_t> bin_index;
    for (const auto& b : r.binaries) {
        bin_index.emplace(b->build_id(), uint16_t(bin_index.size()));
        h.bin_ids.insert(h.bin_ids.end(), b->build_id().bytes().begin(),
                         b->build_id().bytes().end());
        h.symr.push_back(pack_symbols(b->build_id(), b->full_symbols()));
    }
    h.rank_sample_off.push_back(0);
    h.frame_off.push_back(0);
    for (const auto& [rank, stream] : r.samples) {
        h.rank_ids.push_back(rank);
        for (const StackSample& s : stream) {
            h.ts.push_back(s.timestamp_ns);
            for (const FrameRef& f : s.frames) {
                h.pc.push_back(f.offset);
                h.bin.push_back(bin_index.at(f.build_id));
            }
            h.frame_off.push_back(h.pc.size());
        }
        h.rank_sample_off.push_back(h.ts.size());
    }
    for (const CollectiveEvent& e : r.collectives) {
        h.c_rank.push_back(e.rank);
        h.c_group.push_back(e.group);
        h.c_kind.push_back(uint8_t(e.kind));
        h.c_entry.push_back(e.host_entry_ns);
        h.c_exit.push_back(e.host_exit_ns);
        h.c_dur.push_back(e.gpu_duration_ns);
    }
    for (int i = 0; i < r.spec.ranks; ++i) h.group_ranks.push_back(i);
    std::map<std::string, uint32_t> kid;
    for (const GpuEvent& e : r.gpu_events) kid.emplace(e.kernel, 0);
    for (auto& [k, v] : kid) {
        v = uint32_t(h.kernel_names.size());
        h.kernel_names.push_back(k);
    }
    for (const GpuEvent& e : r.gpu_events) {
        h.g_rank.push_back(e.rank);
        h.g_kernel.push_back(kid.at(e.kernel));
        h.g_start.push_back(e.start_ns);
        h.g_dur.push_back(e.duration_ns);
    }
    std::map<std::string, uint32_t> cid;
    for (const OsCounterRecord& o : r.os_counters) {
        for (const auto& [k, v] : o.snapshot.interrupts) cid.emplace(k, 0);
        for (const auto& [k, v] : o.snapshot.softirqs) cid.emplace(k, 0);
    }
    for (auto& [k, v] : cid) {
        v = uint32_t(h.counter_names.size());
        h.counter_names.push_back(k);
    }
    h.o_irq_off.push_back(0);
    h.o_sirq_off.push_back(0);
    for (const OsCounterRecord& o : r.os_counters) {
        h.o_rank.push_back(o.rank);
        h.o_ws.push_back(o.window_start_ns);
        h.o_p50.push_back(o.snapshot.sched_delay_p50_ns);
        h.o_p99.push_back(o.snapshot.sched_delay_p99_ns);
        h.o_mig.push_back(o.snapshot.numa_migrations);
        for (const auto& [k, v] : o.snapshot.interrupts) {
            h.o_irq_key.push_back(cid.at(k));
            h.o_irq_val.push_back(v);
        }
        for (const auto& [k, v] : o.snapshot.softirqs) {
            h.o_sirq_key.push_back(cid.at(k));
            h.o_sirq_val.push_back(v);
        }
        h.o_irq_off.push_back(h.o_irq_key.size());
        h.o_sirq_off.push_back(h.o_sirq_key.size());
    }
    for (const auto& [k, v] : r.baseline.fractions) {
        h.base_names.push_back(k);
        h.base_fracs.push_back(v);
    }
    for (auto& s : h.kernel_names) h.kernel_cstr.push_back(s.c_str());
    for (auto& s : h.counter_names) h.counter_cstr.push_back(s.c_str());
    for (auto& s : h.base_names) h.base_cstr.push_back(s.c_str());

    stg_window& w = h.win;
    w.memory = STG_MEM_HOST;
    w.group = 0;
    w.window_start_ns = r.window_start_ns;
    w.window_end_ns = r.window_end_ns;
    w.max_skew_ns = 50'000'000;  // write_bundle's meta (bundle.cpp:92)
    w.n_ranks = int32_t(h.rank_ids.size());
    w.rank_ids = h.rank_ids.data();
    w.rank_sample_off = h.rank_sample_off.data();
    w.n_bins = int32_t(r.binaries.size());
    w.bin_build_ids = h.bin_ids.data();
    w.n_samples = h.ts.size();
    w.sample_ts = h.ts.data();
    w.sample_frame_off = h.frame_off.data();
    w.n_frames = h.pc.size();
    w.frame_pc = h.pc.data();
    w.frame_bin = h.bin.data();
    w.n_coll = h.c_rank.size();
    w.coll_rank = h.c_rank.data();
    w.coll_group = h.c_group.data();
    w.coll_kind = h.c_kind.data();
    w.coll_entry = h.c_entry.data();
    w.coll_exit = h.c_exit.data();
    w.coll_gpu_dur = h.c_dur.data();
    w.n_group_ranks = int32_t(h.group_ranks.size());
    w.group_ranks = h.group_ranks.data();
    w.n_gpu = h.g_rank.size();
    w.gpu_rank = h.g_rank.data();
    w.gpu_kernel = h.g_kernel.data();
    w.gpu_start = h.g_start.data();
    w.gpu_dur = h.g_dur.data();
    w.n_kernel_names = uint32_t(h.kernel_cstr.size());
    w.kernel_names = h.kernel_cstr.data();
    w.n_os = h.o_rank.size();
    w.os_rank = h.o_rank.data();
    w.os_window_start = h.o_ws.data();
    w.os_p50 = h.o_p50.data();
    w.os_p99 = h.o_p99.data();
    w.os_migrations = h.o_mig.data();
    w.os_irq_off = h.o_irq_off.data();
    w.os_irq_key = h.o_irq_key.data();
    w.os_irq_val = h.o_irq_val.data();
    w.os_sirq_off = h.o_sirq_off.data();
    w.os_sirq_key = h.o_sirq_key.data();
    w.os_sirq_val = h.o_sirq_val.data();
    w.n_counter_names = uint32_t(h.counter_cstr.size());
    w.counter_names = h.counter_cstr.data();
    w.has_baseline = 1;
    w.baseline_delta = r.baseline.delta;
    w.n_baseline = uint32_t(h.base_cstr.size());
    w.baseline_names = h.base_cstr.data();
    w.baseline_fracs = h.base_fracs.data();
    w.has_baseline_iteration = 1;
    w.baseline_iteration_ms = r.baseline_iteration_ms;

    json labels{{"verdict", verdict_name(r.label.expected_verdict)},
                {"affected_ranks", r.label.affected_ranks},
                {"injected_path", r.label.injected_path},
                {"onset_iteration", r.label.onset_iteration}};
    json skews = json::object();
    for (const auto& [rank, skew] : r.injected_skew_ns)
        skews[std::to_string(rank)] = skew;
    labels["injected_skew_ns"] = skews;
    h.labels = labels.dump();
}

// ---------------------------------------------------------- window -> bundle
LoadedBundle to_bundle(const stg_window& w, const fs::path& dir) {
    LoadedBundle b;
    b.dir = dir;
    b.group = w.group;
    b.ranks = w.n_ranks;
    b.max_skew_ns = w.max_skew_ns;
    b.window_start_ns = w.window_start_ns;
    b.window_end_ns = w.window_end_ns;
    for (int32_t i = 0; i < w.n_group_ranks; ++i) b.group_ranks.push_back(w.group_ranks[i]);
    std::vector<BuildId> ids;
    for (int32_t i = 0; i < w.n_bins; ++i) ids.push_back(id_at(w.bin_build_ids + 20 * i));
    for (int32_t ri = 0; ri < w.n_ranks; ++ri) {
        int rank = w.rank_ids[ri];
        std::vector<StackSample>& stream = b.samples[rank];
        for (uint64_t s = w.rank_sample_off[ri]; s < w.rank_sample_off[ri + 1]; ++s) {
            StackSample smp;
            smp.timestamp_ns = w.sample_ts[s];
            smp.rank = rank;
            smp.thread = 0;
            for (uint64_t f = w.sample_frame_off[s]; f < w.sample_frame_off[s + 1]; ++f)
                smp.frames.push_back({ids.at(w.frame_bin[f]), w.frame_pc[f]});
            stream.push_back(std::move(smp));
        }
    }
    for (uint64_t i = 0; i < w.n_coll; ++i)
        b.collectives.push_back({w.coll_rank[i], w.coll_group[i], CollectiveKind(w.coll_kind[i]),
                                 w.coll_entry[i], w.coll_exit[i], w.coll_gpu_dur[i]});
    for (uint64_t i = 0; i < w.n_gpu; ++i)
        b.gpu_events.push_back({w.gpu_rank[i], 0, w.kernel_names[w.gpu_kernel[i]],
                                w.gpu_start[i], w.gpu_dur[i]});
    for (uint64_t i = 0; i < w.n_os; ++i) {
        OsCounterRecord r;
        r.rank = w.os_rank[i];
        r.window_start_ns = w.os_window_start[i];
        r.snapshot.sched_delay_p50_ns = w.os_p50[i];
        r.snapshot.sched_delay_p99_ns = w.os_p99[i];
        r.snapshot.numa_migrations = w.os_migrations[i];
        for (uint64_t k = w.os_irq_off[i]; k < w.os_irq_off[i + 1]; ++k)
            r.snapshot.interrupts[w.counter_names[w.os_irq_key[k]]] = w.os_irq_val[k];
        for (uint64_t k = w.os_sirq_off[i]; k < w.os_sirq_off[i + 1]; ++k)
            r.snapshot.softirqs[w.counter_names[w.os_sirq_key[k]]] = w.os_sirq_val[k];
        b.os_counters.push_back(std::move(r));
    }
    b.baseline.group = w.group;
    b.baseline.epoch = "pre-onset";
    b.baseline.delta = w.has_baseline ? w.baseline_delta : 0.005;
    for (uint32_t i = 0; i < w.n_baseline; ++i)
        b.baseline.fractions[w.baseline_names[i]] = w.baseline_fracs[i];
    b.baseline_iteration_ms = w.has_baseline_iteration ? w.baseline_iteration_ms : 0.0;
    return b;
}

// The reference build_group_data with its per-rank CPU loop (bundle.cpp:289-300)
// fanned out over threads.  Every call is a reference function; the merge keeps
// build_group_data's map semantics, so the GroupData is identical.
//
// shared_cache = true replaces to_folded's per-record symbolization
// (resolve_stack builds a fresh SymbolFile cache for every record, so a
// 1M-entry table is re-parsed per record, symrepo.cpp:99-120) by the
// reference's own resolve_stacks over all records of the rank (one cache per
// call, symrepo.cpp:122-143) followed by fold_symbolized (folded.cpp:73-81).
// That is the same std::map merge of the same resolved names (add_window,
// folded.cpp:21-29, reverses each record to root-first and sums its count into
// the map; fold_symbolized does exactly that), so the folded profile is
// identical — it only makes C2-shaped windows (1M-symbol tables, nearly one
// record per sample) finish in seconds instead of hours.
GroupData build_group_data_threads(const LoadedBundle& bundle, int threads, bool shared_cache = false) {
    GroupData data;
    {
        // Everything except the CPU loop: run the reference itself on a bundle
        // without samples, then add the CPU profiles below.
        LoadedBundle nos = bundle;
        nos.samples.clear();
        data = build_group_data(nos);
    }
    MatchConfig match_cfg{bundle.max_skew_ns};
    auto instances = match_collectives(bundle.collectives, bundle.group_ranks, match_cfg);
    auto offsets = align_clocks(instances);
    std::map<int, int64_t> off = offsets ? *offsets : std::map<int, int64_t>{};
    std::vector<int> ranks;
    for (const auto& [r, s] : bundle.samples) ranks.push_back(r);
    std::vector<std::optional<FoldedProfile>> out(ranks.size());
    std::atomic<size_t> next{0};
    std::vector<std::string> errors(size_t(std::max(threads, 1)));
    auto work = [&](int tid) {
        SymbolRepository repo(bundle.dir);
        try {
            for (size_t i = next++; i < ranks.size(); i = next++) {
                int rank = ranks[i];
                auto it = off.find(rank);
                int64_t o = it == off.end() ? 0 : it->second;
                std::vector<StackSample> in_window;
                for (const StackSample& s : bundle.samples.at(rank))
                    if (s.timestamp_ns - o >= bundle.window_start_ns) in_window.push_back(s);
                if (in_window.empty()) continue;
                auto windows = aggregate_samples(
                    in_window, bundle.window_end_ns - bundle.window_start_ns + 2 * bundle.max_skew_ns);
                if (!shared_cache) {
                    out[i] = to_folded(windows, repo, SymbolFile::LookupMode::ExactRange);
                    continue;
                }
                std::vector<std::vector<FrameRef>> stacks;
                std::vector<uint64_t> counts;
                for (const ProfileWindow& pw : windows)
                    for (const auto& rec : pw.records) {
                        stacks.push_back(rec.frames);
                        counts.push_back(rec.count);
                    }
                auto names = resolve_stacks(stacks, repo, SymbolFile::LookupMode::ExactRange);
                std::vector<std::pair<std::vector<std::string>, uint64_t>> sym;
                sym.reserve(names.size());
                for (size_t k = 0; k < names.size(); ++k) sym.emplace_back(std::move(names[k]), counts[k]);
                if (sym.empty()) throw Error("empty profile window");
                out[i] = fold_symbolized(sym);
            }
        } catch (const std::exception& e) {
            errors[size_t(tid)] = e.what();
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(threads, 1); ++t) pool.emplace_back(work, t);
    for (auto& t : pool) t.join();
    for (const auto& e : errors)
        if (!e.empty()) throw Error(e);
    for (size_t i = 0; i < ranks.size(); ++i)
        if (out[i]) data.cpu_profiles.emplace(ranks[i], std::move(*out[i]));
    return data;
}

json groupdata_json(const GroupData& d) {
    json j;
    j["group"] = d.group;
    json cpu = json::array();
    for (const auto& [rank, p] : d.cpu_profiles) {
        json lines = json::array();
        for (const auto& l : p.lines) lines.push_back(json::array({l.frames, l.count}));
        cpu.push_back({{"rank", rank}, {"total", p.total}, {"lines", lines}});
    }
    j["cpu_profiles"] = cpu;
    json gpu = json::array();
    for (const auto& [rank, g] : d.gpu_profiles) {
        json k = json::array();
        for (const auto& [name, ns] : g.kernel_time_ns) k.push_back(json::array({name, ns}));
        gpu.push_back({{"rank", rank}, {"kernels", k}});
    }
    j["gpu_profiles"] = gpu;
    json os = json::array();
    for (const auto& [rank, s] : d.os_snapshots) {
        json irq = json::array(), sirq = json::array();
        for (const auto& [k, v] : s.interrupts) irq.push_back(json::array({k, v}));
        for (const auto& [k, v] : s.softirqs) sirq.push_back(json::array({k, v}));
        os.push_back({{"rank", rank},
                      {"interrupts", irq},
                      {"softirqs", sirq},
                      {"p50", s.sched_delay_p50_ns},
                      {"p99", s.sched_delay_p99_ns},
                      {"migrations", s.numa_migrations}});
    }
    j["os_snapshots"] = os;
    json lat = json::array();
    for (const auto& inst : d.lateness_per_instance) {
        json row = json::array();
        for (const auto& [r, l] : inst) row.push_back(json::array({r, l}));
        lat.push_back(row);
    }
    j["lateness_per_instance"] = lat;
    j["iteration_times_ms"] = d.iteration_times_ms;
    if (d.baseline) {
        json fr = json::array();
        for (const auto& [k, v] : d.baseline->fractions) fr.push_back(json::array({k, v}));
        j["baseline"] = {{"delta", d.baseline->delta}, {"fractions", fr}};
    } else {
        j["baseline"] = nullptr;
    }
    if (d.baseline_iteration_ms)
        j["baseline_iteration_ms"] = *d.baseline_iteration_ms;
    else
        j["baseline_iteration_ms"] = nullptr;
    return j;
}

char* dup_string(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

fs::path make_repo(const char* tmpdir, int n_symr, const uint8_t* const* symr,
                   const uint64_t* symr_len) {
    fs::path dir = fs::path(tmpdir) /
                   ("strata-ref-" + std::to_string(std::random_device{}()));
    fs::create_directories(dir);
    SymbolRepository repo(dir);
    for (int i = 0; i < n_symr; ++i) {
        std::vector<uint8_t> payload(symr[i], symr[i] + symr_len[i]);
        SymbolFile f = parse_symbols(payload);
        repo.ingest(f.build_id(), payload);
    }
    return dir;
}

}  // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }

void* ref_sim_create(const char* scenario, uint64_t seed, int ranks, int iterations,
                     double sample_rate_hz, double magnitude, int onset_iteration,
                     int analysis_window, char* err, int errcap) {
    try {
        ScenarioSpec spec = default_spec(scenario_from_name(scenario), seed);
        if (ranks > 0) spec.ranks = ranks;
        if (iterations > 0) {
            spec.iterations = iterations;
            // default_spec derives the onset of the all-rank faults from the
            // iteration count (simulate.cpp:296-303); keep it consistent.
            if (spec.onset_iteration != 0) spec.onset_iteration = iterations / 2;
        }
        if (sample_rate_hz > 0) spec.sample_rate_hz = sample_rate_hz;
        if (magnitude > 0) spec.magnitude = magnitude;
        if (onset_iteration >= 0) spec.onset_iteration = onset_iteration;
        if (analysis_window > 0) spec.analysis_window_iterations = analysis_window;
        auto* h = new SimHandle;
        h->res = simulate(spec);
        build_soa(*h);
        return h;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        return nullptr;
    }
}

int ref_sim_window(void* h, stg_window* out) {
    *out = static_cast<SimHandle*>(h)->win;
    return 0;
}
int ref_sim_symr_count(void* h) { return int(static_cast<SimHandle*>(h)->symr.size()); }
int ref_sim_symr(void* h, int i, const uint8_t** p, uint64_t* n) {
    auto* s = static_cast<SimHandle*>(h);
    *p = s->symr.at(size_t(i)).data();
    *n = s->symr.at(size_t(i)).size();
    return 0;
}
const char* ref_sim_labels_json(void* h) { return static_cast<SimHandle*>(h)->labels.c_str(); }
void ref_sim_free(void* h) { delete static_cast<SimHandle*>(h); }

// write_bundle (bundle.cpp:83-164) of a simulation into dir.
int ref_sim_write_bundle(void* h, const char* dir, char* err, int errcap) {
    try {
        write_bundle(static_cast<SimHandle*>(h)->res, dir);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        return 1;
    }
}

// load_bundle alone (bundle.cpp:181-233), timed; returns the sample count.
int ref_bundle_load_time(const char* dir, double* t_load, uint64_t* n_samples, char* err, int errcap) {
    try {
        auto t0 = std::chrono::steady_clock::now();
        LoadedBundle b = load_bundle(dir);
        *t_load = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        uint64_t n = 0;
        for (const auto& [r, s] : b.samples) n += s.size();
        *n_samples = n;
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        return 1;
    }
}

// load_bundle + build_group_data + diagnose on a bundle directory, timed per stage.
int ref_bundle_run(const char* dir, int want_json, char** out_json, double* t_load, double* t_build,
                   double* t_diag, char* err, int errcap) {
    try {
        auto t0 = std::chrono::steady_clock::now();
        LoadedBundle b = load_bundle(dir);
        auto t1 = std::chrono::steady_clock::now();
        GroupData data = build_group_data(b);
        auto t2 = std::chrono::steady_clock::now();
        DiagnosisReport rep = diagnose(data);
        auto t3 = std::chrono::steady_clock::now();
        if (t_load) *t_load = std::chrono::duration<double>(t1 - t0).count();
        if (t_build) *t_build = std::chrono::duration<double>(t2 - t1).count();
        if (t_diag) *t_diag = std::chrono::duration<double>(t3 - t2).count();
        if (out_json) {
            json j;
            if (want_json) j["groupdata"] = groupdata_json(data);
            j["report"] = json::parse(rep.to_json());
            *out_json = dup_string(j.dump());
        }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        return 1;
    }
}

// build_group_data + diagnose on the reference.  threads <= 1 runs the
// reference build_group_data as-is (single-threaded, the reference's only
// mode); threads > 1 uses the rank-parallel harness above.
// shared_cache = 1: the CPU loop symbolizes through resolve_stacks (see
// build_group_data_threads) — same GroupData, C2-shaped windows feasible.
int ref_window_run_ex(const stg_window* w, int n_symr, const uint8_t* const* symr,
                      const uint64_t* symr_len, const char* tmpdir, int threads, int shared_cache,
                      int want_json, char** out_json, double* t_build, double* t_diag,
                      char* err, int errcap) {
    fs::path dir;
    try {
        dir = make_repo(tmpdir, n_symr, symr, symr_len);
        LoadedBundle b = to_bundle(*w, dir);
        auto t0 = std::chrono::steady_clock::now();
        GroupData data = (threads > 1 || shared_cache) ? build_group_data_threads(b, std::max(threads, 1), shared_cache != 0)
                                                       : build_group_data(b);
        auto t1 = std::chrono::steady_clock::now();
        DiagnosisReport rep = diagnose(data);
        auto t2 = std::chrono::steady_clock::now();
        if (t_build) *t_build = std::chrono::duration<double>(t1 - t0).count();
        if (t_diag) *t_diag = std::chrono::duration<double>(t2 - t1).count();
        if (out_json) {
            json j;
            if (want_json) j["groupdata"] = groupdata_json(data);
            j["report"] = json::parse(rep.to_json());
            j["report_json_raw"] = rep.to_json();  // the reference's own bytes
            j["report_text"] = rep.to_text();
            if (want_json == 2) {
                // the text artifacts of `strata diagnose` / `strata flamegraph`
                // (tools/strata.cpp:97-131): every rank's folded text, each
                // flagged rank's diff against the reference rank, and the diff
                // of the first two profiled ranks both ways
                json folded = json::array(), diffs = json::array();
                std::vector<int> ranks;
                for (const auto& [rank, prof] : data.cpu_profiles) {
                    folded.push_back(json::array({rank, prof.to_string()}));
                    ranks.push_back(rank);
                }
                auto add_diff = [&](int a, int b) {
                    diffs.push_back(json::array(
                        {a, b, diff_folded(data.cpu_profiles.at(a), data.cpu_profiles.at(b))}));
                };
                if (rep.reference_rank && data.cpu_profiles.count(*rep.reference_rank))
                    for (int r : rep.flagged_ranks)
                        if (data.cpu_profiles.count(r)) add_diff(r, *rep.reference_rank);
                if (ranks.size() >= 2) {
                    add_diff(ranks[0], ranks[1]);
                    add_diff(ranks[1], ranks[0]);
                }
                if (!ranks.empty()) add_diff(ranks[0], ranks[0]);
                // flame graphs (svg.cpp:157-172) with the CLI's titles (tools/strata.cpp:119-148)
                json svgs = json::array(), svg_diffs = json::array();
                for (size_t q = 0; q < ranks.size() && q < 6; ++q) {
                    SvgOptions o;
                    o.title = "rank " + std::to_string(ranks[q]);
                    svgs.push_back(json::array({ranks[q], render_flamegraph(data.cpu_profiles.at(ranks[q]), o)}));
                }
                auto add_svg_diff = [&](int a, int b) {
                    SvgOptions o;
                    o.title = "rank " + std::to_string(a) + " vs rank " + std::to_string(b);
                    svg_diffs.push_back(json::array(
                        {a, b, render_diff_flamegraph(data.cpu_profiles.at(a), data.cpu_profiles.at(b), o)}));
                };
                if (rep.reference_rank && data.cpu_profiles.count(*rep.reference_rank))
                    for (int r : rep.flagged_ranks)
                        if (data.cpu_profiles.count(r)) add_svg_diff(r, *rep.reference_rank);
                if (ranks.size() >= 2) add_svg_diff(ranks[0], ranks[1]);
                j["artifacts"] = {{"folded", folded}, {"diffs", diffs}, {"svg", svgs}, {"svg_diffs", svg_diffs}};
            }
            *out_json = dup_string(j.dump());
        }
        fs::remove_all(dir);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        if (!dir.empty()) fs::remove_all(dir);
        return 1;
    }
}

int ref_window_run(const stg_window* w, int n_symr, const uint8_t* const* symr,
                   const uint64_t* symr_len, const char* tmpdir, int threads,
                   int want_json, char** out_json, double* t_build, double* t_diag,
                   char* err, int errcap) {
    return ref_window_run_ex(w, n_symr, symr, symr_len, tmpdir, threads, 0, want_json, out_json, t_build, t_diag,
                             err, errcap);
}

// ---- single verbs, for unit parity ----------------------------------------

// SymbolFile::lookup (symfile.cpp:54-75) over one SYMR payload; out_idx gets the
// entry index (or -1) and probes the bisection probe count.
int ref_lookup(const uint8_t* symr, uint64_t len, uint64_t n, const uint64_t* offs,
               int mode, int64_t* out_idx, uint64_t* probes, char* err, int errcap) {
    try {
        SymbolFile f = parse_symbols(std::vector<uint8_t>(symr, symr + len));
        const auto& e = f.entries();
        for (uint64_t i = 0; i < n; ++i) {
            uint64_t p = 0;
            auto name = f.lookup(offs[i], SymbolFile::LookupMode(mode), &p);
            if (probes) probes[i] = p;
            if (!name) {
                out_idx[i] = -1;
                continue;
            }
            // Recover the entry index: greatest start <= offset.
            auto it = std::upper_bound(e.begin(), e.end(), offs[i],
                                       [](uint64_t v, const SymbolEntry& s) { return v < s.start; });
            out_idx[i] = int64_t(it - e.begin()) - 1;
        }
        return 0;
    } catch (const std::exception& ex) {
        set_err(err, errcap, ex.what());
        return 1;
    }
}

// parse_symbols validation (symfile.cpp:117-157): 0 if accepted, else message.
int ref_parse_symbols(const uint8_t* symr, uint64_t len, char* err, int errcap) {
    try {
        parse_symbols(std::vector<uint8_t>(symr, symr + len));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        return 1;
    }
}

// pack_symbols (symfile.cpp:77-115) from SoA entries; names are NUL-separated.
int ref_pack_symbols(const uint8_t* build_id, uint64_t n, const uint64_t* starts,
                     const uint32_t* sizes, const char* names_blob, uint8_t** out,
                     uint64_t* out_len, char* err, int errcap) {
    try {
        std::vector<SymbolEntry> es;
        const char* p = names_blob;
        for (uint64_t i = 0; i < n; ++i) {
            std::string name(p);
            p += name.size() + 1;
            es.push_back({starts[i], sizes[i], name});
        }
        auto bytes = pack_symbols(id_at(build_id), es);
        *out = static_cast<uint8_t*>(std::malloc(bytes.size()));
        std::memcpy(*out, bytes.data(), bytes.size());
        *out_len = bytes.size();
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        return 1;
    }
}

// aggregate_samples (samples.cpp:31-85) on a raw SoA stream.  Output JSON:
// {"windows": [[rank, start, end, [[first_sample, count], ...]], ...]} where
// first_sample is the stream index of the first sample whose frames equal the
// record's (found by scanning the window's samples in order).
int ref_aggregate_samples(uint64_t n, const int64_t* ts, const int32_t* rank, const uint64_t* foff,
                          const uint64_t* pc, const uint16_t* bin, int n_bins, const uint8_t* bin_ids,
                          int64_t drain, char** out_json, double* t_agg, char* err, int errcap) {
    try {
        std::vector<BuildId> ids;
        for (int i = 0; i < n_bins; ++i) ids.push_back(id_at(bin_ids + 20 * i));
        std::vector<StackSample> stream(n);
        for (uint64_t i = 0; i < n; ++i) {
            stream[i].timestamp_ns = ts[i];
            stream[i].rank = rank ? rank[i] : 0;
            for (uint64_t f = foff[i]; f < foff[i + 1]; ++f) stream[i].frames.push_back({ids.at(bin[f]), pc[f]});
        }
        auto t0 = std::chrono::steady_clock::now();
        std::vector<ProfileWindow> wins = aggregate_samples(stream, drain);
        if (t_agg) *t_agg = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (!out_json) return 0;
        json out = json::array();
        uint64_t cur = 0;
        for (const ProfileWindow& w : wins) {
            while (cur < n && stream[cur].timestamp_ns < w.window_start_ns) ++cur;
            std::vector<std::pair<const std::vector<FrameRef>*, uint64_t>> first;
            uint64_t e = cur;
            while (e < n && stream[e].timestamp_ns < w.window_end_ns) ++e;
            json recs = json::array();
            for (const auto& r : w.records) {
                uint64_t f = e;
                for (uint64_t i = cur; i < e; ++i)
                    if (stream[i].frames == r.frames) { f = i; break; }
                recs.push_back(json::array({f, r.count}));
            }
            out.push_back(json::array({w.rank, w.window_start_ns, w.window_end_ns, recs}));
            cur = e;
        }
        *out_json = dup_string(json{{"windows", out}}.dump());
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        return 1;
    }
}

// unknown_frame_label (symfile.cpp:159-163)
int ref_unknown_label(const uint8_t* build_id, uint64_t off, char* buf, int cap) {
    std::string s = unknown_frame_label(id_at(build_id), off);
    std::snprintf(buf, size_t(cap), "%s", s.c_str());
    return int(s.size());
}

// BuildId::digest (SHA-1, build_id.cpp:96-105) — used to derive test build ids
// exactly like the reference tests do (BuildId::digest(std::string(1, c))).
void ref_digest(const uint8_t* data, uint64_t len, uint8_t* out20) {
    BuildId id = BuildId::digest(std::string_view(reinterpret_cast<const char*>(data), len));
    std::memcpy(out20, id.bytes().data(), 20);
}

// match_collectives -> align_clocks -> entry_lateness over a flat event list
// (collective.cpp:29-142).  Output JSON: instances (group, kind, partial,
// events[[rank, entry, exit]]), offsets (or null), lateness per complete inst.
int ref_collectives(uint64_t n, const int32_t* rank, const int32_t* group,
                    const uint8_t* kind, const int64_t* entry, const int64_t* exit_,
                    const int64_t* dur, int32_t n_group_ranks, const int32_t* group_ranks,
                    int64_t max_skew, char** out_json, char* err, int errcap) {
    try {
        std::vector<CollectiveEvent> ev;
        for (uint64_t i = 0; i < n; ++i)
            ev.push_back({rank[i], group[i], CollectiveKind(kind[i]), entry[i], exit_[i], dur[i]});
        std::vector<int> gr(group_ranks, group_ranks + n_group_ranks);
        auto inst = match_collectives(ev, gr, MatchConfig{max_skew});
        auto off = align_clocks(inst);
        json j;
        json arr = json::array();
        for (const auto& c : inst) {
            json es = json::array();
            for (const auto& [r, e] : c.events)
                es.push_back(json::array({r, e.host_entry_ns, e.host_exit_ns}));
            json o{{"group", c.group}, {"kind", int(c.kind)}, {"partial", c.partial}, {"events", es}};
            if (!c.partial) {
                json lat = json::array();
                for (const auto& [r, l] : entry_lateness(c, off ? *off : std::map<int, int64_t>{}))
                    lat.push_back(json::array({r, l}));
                o["lateness"] = lat;
            }
            arr.push_back(o);
        }
        j["instances"] = arr;
        if (off) {
            json o = json::array();
            for (const auto& [r, v] : *off) o.push_back(json::array({r, v}));
            j["offsets"] = o;
        } else {
            j["offsets"] = nullptr;
        }
        *out_json = dup_string(j.dump());
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        return 1;
    }
}

// detect_straggler (diagnosis.cpp:76-111) over a dense I x R lateness matrix
// (NaN = rank absent from the instance).
int ref_detect_straggler(uint64_t n_inst, int32_t n_ranks, const int32_t* ranks,
                         const double* lat, double k, char** out_json, char* err, int errcap) {
    try {
        std::vector<std::map<int, double>> per;
        for (uint64_t i = 0; i < n_inst; ++i) {
            std::map<int, double> m;
            for (int32_t r = 0; r < n_ranks; ++r) {
                double v = lat[i * uint64_t(n_ranks) + uint64_t(r)];
                if (v == v) m[ranks[r]] = v;
            }
            per.push_back(std::move(m));
        }
        auto alerts = detect_straggler(per, 0, k);
        json arr = json::array();
        for (const auto& a : alerts)
            arr.push_back({{"rank", a.rank},
                           {"mean_lateness_ms", a.mean_lateness_ms},
                           {"z_score", a.z_score},
                           {"flagged_instances", a.flagged_instances},
                           {"window_instances", a.window_instances}});
        *out_json = dup_string(arr.dump());
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        return 1;
    }
}

// compute_waterline + flag_ranks (diagnosis.cpp:35-71) over the CPU profiles
// the reference builds for a window.
int ref_waterline(const stg_window* w, int n_symr, const uint8_t* const* symr,
                  const uint64_t* symr_len, const char* tmpdir, double k, char** out_json,
                  char* err, int errcap) {
    fs::path dir;
    try {
        dir = make_repo(tmpdir, n_symr, symr, symr_len);
        LoadedBundle b = to_bundle(*w, dir);
        GroupData data = build_group_data(b);
        Waterline wl = compute_waterline(data.cpu_profiles, data.group, 100, k);
        auto flags = flag_ranks(wl, data.cpu_profiles);
        json fn = json::array();
        for (const auto& [name, st] : wl.functions)
            fn.push_back(json::array({name, st.mean, st.stddev}));
        json fl = json::array();
        for (const auto& f : flags)
            fl.push_back(json::array({f.rank, f.function, f.fraction, f.threshold}));
        json fr = json::array();
        for (const auto& [rank, p] : data.cpu_profiles) {
            json row = json::array();
            for (const auto& [name, v] : p.inclusive_fractions()) row.push_back(json::array({name, v}));
            fr.push_back({{"rank", rank}, {"fractions", row}});
        }
        *out_json = dup_string(json{{"functions", fn}, {"flags", fl}, {"fractions", fr}}.dump());
        fs::remove_all(dir);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errcap, e.what());
        if (!dir.empty()) fs::remove_all(dir);
        return 1;
    }
}

}  // extern "C"
