// stg_bundle_host.cpp — load_bundle (proj/core/src/bundle.cpp:181-233) for the
// analysis path: meta.json, gpu_events.jsonl and os_counters.jsonl (small) are
// parsed on the host with nlohmann::json 3.11 — the parser the reference uses,
// so their errors carry the same text; samples.jsonl and collectives.jsonl (the
// bulk) are decoded on the GPU (stg_bundle.cu).  The symbol tables of the
// bundle's binaries are ingested from its repository
// (<dir>/symbols/<hex[0:2]>/<hex>.symr, symrepo.cpp:14-17), as build_group_data
// would load them on demand.
#include <chrono>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>

#include "bundle.h"
#include "json.hpp"

namespace stg {

namespace fs = std::filesystem;
using nlohmann::json;

namespace {

// read_file (bundle.cpp:24-30)
std::string read_file(const fs::path& p) {
    std::ifstream in(p, std::ios::binary);
    if (!in) fail(STG_EINVAL, "missing bundle file: " + p.string());
    std::string s;
    in.seekg(0, std::ios::end);
    s.resize(size_t(in.tellg()));
    in.seekg(0);
    in.read(s.data(), std::streamsize(s.size()));
    return s;
}

template <class F>
void for_lines(const std::string& text, F&& f) {
    std::istringstream is(text);
    for (std::string line; std::getline(is, line);) {
        if (line.empty()) continue;
        f(json::parse(line));
    }
}

double secs(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

void bundle_load(Ctx& c, const std::string& dir_s, stg_bundle_info* info) {
    const auto t0 = std::chrono::steady_clock::now();
    auto bp = std::make_shared<Bundle>();
    Bundle& b = *bp;
    const fs::path dir(dir_s);
    try {
        // meta.json (bundle.cpp:185-201)
        json meta = json::parse(read_file(dir / "meta.json"));
        b.scenario = meta.at("scenario").get<std::string>();
        (void)meta.at("seed").get<uint64_t>();
        (void)meta.at("ranks").get<int>();
        b.w.group = meta.at("group").get<int>();
        b.group_ranks = meta.at("group_ranks").get<std::vector<int32_t>>();
        b.w.max_skew_ns = meta.at("max_skew_ns").get<int64_t>();
        b.w.window_start_ns = meta.at("window_start_ns").get<int64_t>();
        b.w.window_end_ns = meta.at("window_end_ns").get<int64_t>();
        const json& base = meta.at("baseline");
        (void)base.at("epoch").get<std::string>();
        b.w.baseline_delta = base.at("delta").get<double>();
        for (const auto& [k, v] : base.at("fractions").get<std::map<std::string, double>>()) {
            b.base_names.push_back(k);
            b.base_fracs.push_back(v);
        }
        b.w.baseline_iteration_ms = base.at("iteration_ms").get<double>();
    } catch (const json::exception& e) {
        fail(STG_EINVAL, e.what());
    }
    // bulk files: pipelined read -> device, then decoded on the GPU
    double t_read = 0, t_dec = 0;
    uint64_t bytes_s = 0, bytes_c = 0;
    auto tr = std::chrono::steady_clock::now();
    const uint8_t* ds = upload_file(c, (dir / "samples.jsonl").string(), "bs", bytes_s);
    t_read += secs(tr);
    auto td = std::chrono::steady_clock::now();
    bundle_decode_samples(c, ds, bytes_s, b.bulk);
    t_dec += secs(td);
    tr = std::chrono::steady_clock::now();
    const uint8_t* dc = upload_file(c, (dir / "collectives.jsonl").string(), "bc", bytes_c);
    t_read += secs(tr);
    td = std::chrono::steady_clock::now();
    bundle_decode_collectives(c, dc, bytes_c, b.bulk);
    t_dec += secs(td);
    try {
        // gpu_events.jsonl (bundle.cpp:216-225): kernels interned in name order
        std::vector<std::string> kern;
        std::map<std::string, uint32_t> kid;
        for_lines(read_file(dir / "gpu_events.jsonl"), [&](const json& j) {
            b.g_rank.push_back(j.at("rank").get<int>());
            (void)j.at("iter").get<int>();
            kern.push_back(j.at("kernel").get<std::string>());
            b.g_start.push_back(j.at("start").get<int64_t>());
            b.g_dur.push_back(j.at("dur").get<int64_t>());
            kid.emplace(kern.back(), 0);
        });
        for (auto& [k, v] : kid) {
            v = uint32_t(b.kernel_names.size());
            b.kernel_names.push_back(k);
        }
        for (const auto& k : kern) b.g_kernel.push_back(kid.at(k));
        // os_counters.jsonl (bundle.cpp:226-230, os_from_json :68-80)
        std::vector<std::map<std::string, int64_t>> irq, sirq;
        for_lines(read_file(dir / "os_counters.jsonl"), [&](const json& j) {
            b.o_rank.push_back(j.at("rank").get<int>());
            b.o_ws.push_back(j.at("window_start").get<int64_t>());
            irq.push_back(j.at("interrupts").get<std::map<std::string, int64_t>>());
            sirq.push_back(j.at("softirqs").get<std::map<std::string, int64_t>>());
            b.o_p50.push_back(j.at("sched_delay_p50_ns").get<int64_t>());
            b.o_p99.push_back(j.at("sched_delay_p99_ns").get<int64_t>());
            b.o_mig.push_back(j.at("numa_migrations").get<int64_t>());
        });
        std::map<std::string, uint32_t> cid;
        for (size_t i = 0; i < irq.size(); ++i) {
            for (const auto& [k, v] : irq[i]) cid.emplace(k, 0);
            for (const auto& [k, v] : sirq[i]) cid.emplace(k, 0);
        }
        for (auto& [k, v] : cid) {
            v = uint32_t(b.counter_names.size());
            b.counter_names.push_back(k);
        }
        for (size_t i = 0; i < irq.size(); ++i) {
            for (const auto& [k, v] : irq[i]) {
                b.irq_k.push_back(cid.at(k));
                b.irq_v.push_back(v);
            }
            for (const auto& [k, v] : sirq[i]) {
                b.sirq_k.push_back(cid.at(k));
                b.sirq_v.push_back(v);
            }
            b.irq_off.push_back(b.irq_k.size());
            b.sirq_off.push_back(b.sirq_k.size());
        }
    } catch (const json::exception& e) {
        fail(STG_EINVAL, e.what());
    }
    // symbol tables of the referenced binaries (SymbolRepository::path_for)
    uint32_t ingested = 0;
    const size_t nb = b.bulk.bin_ids.size() / 20;
    for (size_t i = 0; i < nb; ++i) {
        const uint8_t* id = b.bulk.bin_ids.data() + 20 * i;
        const std::string hex = hex_id(id);
        const fs::path p = dir / "symbols" / hex.substr(0, 2) / (hex + ".symr");
        std::ifstream in(p, std::ios::binary);
        if (!in) continue;
        std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        int stored = 0;
        symtab_ingest(c, id, reinterpret_cast<const uint8_t*>(bytes.data()), bytes.size(), &stored);
        ingested += uint32_t(stored);
    }
    // the window (LoadedBundle as build_group_data reads it, bundle.cpp:252-324)
    for (auto& s : b.kernel_names) b.kernel_cstr.push_back(s.c_str());
    for (auto& s : b.counter_names) b.counter_cstr.push_back(s.c_str());
    for (auto& s : b.base_names) b.base_cstr.push_back(s.c_str());
    stg_window& w = b.w;
    const BundleBulk& k = b.bulk;
    w.memory = STG_MEM_DEVICE;
    w.n_ranks = int32_t(k.rank_ids.size());
    w.rank_ids = k.rank_ids.data();
    w.rank_sample_off = k.rank_sample_off.data();
    w.n_bins = int32_t(nb);
    w.bin_build_ids = k.bin_ids.data();
    w.n_samples = k.n_samples;
    w.sample_ts = k.ts;
    w.sample_frame_off = k.foff;
    w.n_frames = k.n_frames;
    w.frame_pc = k.pc;
    w.frame_bin = k.bin;
    w.coll_memory = STG_MEM_DEVICE;
    w.side_memory = STG_MEM_HOST;  // gpu/os records are decoded on the host
    w.n_coll = k.n_coll;
    w.coll_rank = k.c_rank;
    w.coll_group = k.c_group;
    w.coll_kind = k.c_kind;
    w.coll_entry = k.c_entry;
    w.coll_exit = k.c_exit;
    w.coll_gpu_dur = k.c_dur;
    w.n_group_ranks = int32_t(b.group_ranks.size());
    w.group_ranks = b.group_ranks.data();
    w.n_gpu = b.g_rank.size();
    w.gpu_rank = b.g_rank.data();
    w.gpu_kernel = b.g_kernel.data();
    w.gpu_start = b.g_start.data();
    w.gpu_dur = b.g_dur.data();
    w.n_kernel_names = uint32_t(b.kernel_cstr.size());
    w.kernel_names = b.kernel_cstr.data();
    w.n_os = b.o_rank.size();
    w.os_rank = b.o_rank.data();
    w.os_window_start = b.o_ws.data();
    w.os_p50 = b.o_p50.data();
    w.os_p99 = b.o_p99.data();
    w.os_migrations = b.o_mig.data();
    w.os_irq_off = b.irq_off.data();
    w.os_irq_key = b.irq_k.data();
    w.os_irq_val = b.irq_v.data();
    w.os_sirq_off = b.sirq_off.data();
    w.os_sirq_key = b.sirq_k.data();
    w.os_sirq_val = b.sirq_v.data();
    w.n_counter_names = uint32_t(b.counter_cstr.size());
    w.counter_names = b.counter_cstr.data();
    // LoadedBundle always carries its baseline (bundle.cpp:196-201, 256-257)
    w.has_baseline = 1;
    w.n_baseline = uint32_t(b.base_cstr.size());
    w.baseline_names = b.base_cstr.data();
    w.baseline_fracs = b.base_fracs.data();
    w.has_baseline_iteration = 1;
    stg_bundle_info& in = b.info;
    in.n_ranks = uint32_t(k.rank_ids.size());
    in.n_bins = uint32_t(nb);
    in.n_tables_ingested = ingested;
    in.n_samples = k.n_samples;
    in.n_frames = k.n_frames;
    in.n_coll = k.n_coll;
    in.n_gpu = b.g_rank.size();
    in.n_os = b.o_rank.size();
    in.bulk_bytes = bytes_s + bytes_c;
    in.read_s = t_read;
    in.decode_s = t_dec;
    in.total_s = secs(t0);
    c.bundle = bp;
    if (info) *info = in;
}

}  // namespace stg
