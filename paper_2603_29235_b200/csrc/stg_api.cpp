// stg_api.cpp — the extern "C" surface of libstg (include/stg.h).  Every entry
// point catches stg::Error / std::exception, stores the message thread-locally
// and returns a status code; no C++ exception crosses the boundary.
#include <cstring>
#include <string>

#include <nccl.h>

#include "bundle.h"
#include "result.h"
#include "stg_internal.h"

namespace stg {
void window_run(Ctx& c, const stg_window& w, const stg_config& cfg);
std::string groupdata_json(Ctx& c, uint32_t parts);
std::string report_json(Ctx& c);
std::string report_text_of(Ctx& c);
std::string flamegraph_svg(Ctx& c, int kind, int32_t rank_a, int32_t rank_b, const stg_svg_options& o);
std::string waterline_json(Ctx& c);
void run_resolve(Ctx& c, Result& res, uint64_t n, const uint64_t* pc, const uint16_t* bin, int32_t n_bins,
                 const uint8_t* ids, int mode, uint32_t* out);
void rank_lines(Ctx& c, uint32_t i, std::vector<uint64_t>& key_off, std::vector<uint32_t>& keys,
                std::vector<uint64_t>& counts);
uint64_t render_folded(Ctx& c, int kind, int32_t rank_a, int32_t rank_b);
void aggregate_samples(Ctx& c, const stg_stream& in, int64_t drain, int flags, uint64_t* n_windows,
                       uint64_t* n_records);
void aggregate_windows(Ctx& c, int64_t* start, int64_t* end, uint64_t* rec_off);
void aggregate_records(Ctx& c, uint64_t* first_sample, uint64_t* count);
void render_copy(Ctx& c, char* buf, uint64_t len);
}  // namespace stg

struct stg_ctx {
    stg::Ctx impl;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_err.clear();
        return STG_OK;
    } catch (const stg::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return STG_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return STG_EINVAL;
    }
}

int copy_out(const std::string& s, char* buf, uint64_t cap, uint64_t* needed) {
    if (needed) *needed = s.size() + 1;
    if (!buf) return STG_OK;
    if (cap < s.size() + 1) {
        g_err = "buffer too small";
        return STG_EINVAL;
    }
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return STG_OK;
}

stg::Result& need_result(stg_ctx* c) {
    if (!c->impl.result) stg::fail(STG_ESTATE, "no window result on this context");
    return *c->impl.result;
}
}  // namespace

extern "C" {

const char* stg_last_error(void) { return g_err.c_str(); }
int stg_abi_version(void) { return STG_ABI_VERSION; }

void stg_abi_sizes(uint64_t* window, uint64_t* config, uint64_t* stats) {
    if (window) *window = sizeof(stg_window);
    if (config) *config = sizeof(stg_config);
    if (stats) *stats = sizeof(stg_run_stats);
}

int stg_create(int device, stg_ctx** out) {
    return guard([&] {
        int n = 0;
        STG_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) stg::fail(STG_EINVAL, "no such CUDA device");
        STG_CUDA(cudaSetDevice(device));
        auto* c = new stg_ctx;
        c->impl.device = device;
        cudaError_t e = cudaStreamCreateWithFlags(&c->impl.stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete c;
            stg::fail(STG_ECUDA, cudaGetErrorString(e));
        }
        *out = c;
    });
}

void stg_destroy(stg_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->impl.device);
    if (ctx->impl.comm) ncclCommDestroy(static_cast<ncclComm_t>(ctx->impl.comm));
    delete ctx;
}

int stg_dist_unique_id(uint8_t id[128]) {
    return guard([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId u;
        ncclResult_t r = ncclGetUniqueId(&u);
        if (r != ncclSuccess) stg::fail(STG_ECUDA, std::string("NCCL: ") + ncclGetErrorString(r));
        std::memcpy(id, &u, 128);
    });
}

int stg_dist_init(stg_ctx* ctx, int world_size, int world_rank, const uint8_t id[128]) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        if (world_size < 1 || world_rank < 0 || world_rank >= world_size) stg::fail(STG_EINVAL, "bad world size/rank");
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        if (ctx->impl.comm) {
            ncclCommDestroy(static_cast<ncclComm_t>(ctx->impl.comm));
            ctx->impl.comm = nullptr;
        }
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        ncclComm_t comm;
        ncclResult_t r = ncclCommInitRank(&comm, world_size, u, world_rank);
        if (r != ncclSuccess) stg::fail(STG_ECUDA, std::string("NCCL: ") + ncclGetErrorString(r));
        ctx->impl.comm = comm;
        ctx->impl.world = world_size;
        ctx->impl.wrank = world_rank;
    });
}

int stg_symtab_ingest(stg_ctx* ctx, const uint8_t* claimed_id, const uint8_t* symr, uint64_t len, int* stored) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        stg::symtab_ingest(ctx->impl, claimed_id, symr, len, stored);
    });
}

int stg_symtab_count(stg_ctx* ctx, uint32_t* n) {
    return guard([&] { *n = uint32_t(ctx->impl.tables.size()); });
}

int stg_resolve(stg_ctx* ctx, uint64_t n_frames, const uint64_t* frame_pc, const uint16_t* frame_bin,
                int32_t n_bins, const uint8_t* bin_build_ids, int mode, uint32_t* out_keys) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        if (mode != STG_LOOKUP_EXACT_RANGE && mode != STG_LOOKUP_NEAREST_LOWER) stg::fail(STG_EINVAL, "bad lookup mode");
        if (!ctx->impl.result) ctx->impl.result = std::make_unique<stg::Result>();
        stg::run_resolve(ctx->impl, *ctx->impl.result, n_frames, frame_pc, frame_bin, n_bins, bin_build_ids, mode,
                         out_keys);
    });
}

int stg_name(stg_ctx* ctx, uint32_t key, char* buf, uint64_t cap, uint64_t* needed) {
    std::string s;
    int rc = guard([&] {
        stg::Result& r = need_result(ctx);
        if (!r.dict || key >= r.n_names) stg::fail(STG_EINVAL, "name key out of range");
        s = r.name_of(key);
    });
    if (rc) return rc;
    return copy_out(s, buf, cap, needed);
}

int stg_name_count(stg_ctx* ctx, uint32_t* n) {
    return guard([&] { *n = uint32_t(need_result(ctx).n_names); });
}

void stg_config_default(stg_config* c) {
    std::memset(c, 0, sizeof *c);
    c->window_iterations = 100;
    c->k = 2.0;
    c->delta = 0.005;
    c->iteration_regression_gate = 0.03;
    c->gpu_median_uniform = 0.03;
    c->gpu_cv_uniform = 0.25;
    c->gpu_top_share_specific = 0.60;
    c->gpu_median_none = 0.01;
    c->gpu_ref_floor_ns = 1000000;
    std::strcpy(c->gpu_exclude_prefix, "nccl");
    c->os_min_ratio = 2.0;
    c->os_interrupt_floor = 1000;
    c->os_sched_delay_floor_ns = 1000000;
    c->os_migration_floor = 100;
    c->lookup_mode = STG_LOOKUP_EXACT_RANGE;
    c->want_waterline = 0;
    c->verify = 0;
    c->debug_weak_prefix_key = 0;
}

int stg_window_run(stg_ctx* ctx, const stg_window* win, const stg_config* cfg, stg_run_stats* stats) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        stg_config def;
        stg_config_default(&def);
        stg::window_run(ctx->impl, *win, cfg ? *cfg : def);
        if (stats) *stats = ctx->impl.result->stats;
    });
}

int stg_result_groupdata_json(stg_ctx* ctx, char* buf, uint64_t cap, uint64_t* needed) {
    std::string s;
    int rc = guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        need_result(ctx);
        s = stg::groupdata_json(ctx->impl, STG_GD_ALL);
    });
    if (rc) return rc;
    return copy_out(s, buf, cap, needed);
}

int stg_result_groupdata_json_parts(stg_ctx* ctx, uint32_t parts, char* buf, uint64_t cap, uint64_t* needed) {
    std::string s;
    int rc = guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        need_result(ctx);
        s = stg::groupdata_json(ctx->impl, parts);
    });
    if (rc) return rc;
    return copy_out(s, buf, cap, needed);
}

int stg_result_report_json(stg_ctx* ctx, char* buf, uint64_t cap, uint64_t* needed) {
    std::string s;
    int rc = guard([&] {
        need_result(ctx);
        s = stg::report_json(ctx->impl);
    });
    if (rc) return rc;
    return copy_out(s, buf, cap, needed);
}

int stg_result_report_text(stg_ctx* ctx, char* buf, uint64_t cap, uint64_t* needed) {
    std::string s;
    int rc = guard([&] {
        need_result(ctx);
        s = stg::report_text_of(ctx->impl);
    });
    if (rc) return rc;
    return copy_out(s, buf, cap, needed);
}

int stg_result_waterline_json(stg_ctx* ctx, char* buf, uint64_t cap, uint64_t* needed) {
    std::string s;
    int rc = guard([&] {
        stg::Result& r = need_result(ctx);
        if (!r.waterline_done) stg::fail(STG_ESTATE, "run the window with want_waterline = 1");
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        s = stg::waterline_json(ctx->impl);
    });
    if (rc) return rc;
    return copy_out(s, buf, cap, needed);
}

int stg_result_rank_count(stg_ctx* ctx, uint32_t* n) {
    return guard([&] { *n = uint32_t(need_result(ctx).cpu_rank_ids.size()); });
}

int stg_result_rank_info(stg_ctx* ctx, uint32_t i, int32_t* rank, uint64_t* n_lines, uint64_t* total,
                         uint64_t* n_keys) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        stg::Result& r = need_result(ctx);
        if (i >= r.cpu_rank_ids.size()) stg::fail(STG_ESTATE, "rank index out of range");
        std::vector<uint64_t> ko, cnt;
        std::vector<uint32_t> keys;
        stg::rank_lines(ctx->impl, i, ko, keys, cnt);
        if (rank) *rank = r.cpu_rank_ids[i];
        if (n_lines) *n_lines = cnt.size();
        if (total) *total = r.cpu_totals[i];
        if (n_keys) *n_keys = keys.size();
    });
}

int stg_result_rank_lines(stg_ctx* ctx, uint32_t i, uint64_t* line_key_off, uint32_t* keys_out, uint64_t* counts) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        stg::Result& r = need_result(ctx);
        if (i >= r.cpu_rank_ids.size()) stg::fail(STG_ESTATE, "rank index out of range");
        std::vector<uint64_t> ko, cnt;
        std::vector<uint32_t> keys;
        stg::rank_lines(ctx->impl, i, ko, keys, cnt);
        std::memcpy(line_key_off, ko.data(), ko.size() * sizeof(uint64_t));
        std::memcpy(keys_out, keys.data(), keys.size() * sizeof(uint32_t));
        std::memcpy(counts, cnt.data(), cnt.size() * sizeof(uint64_t));
    });
}

static int folded_text(stg_ctx* ctx, int kind, int32_t a, int32_t b, char* buf, uint64_t cap, uint64_t* needed) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        need_result(ctx);
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        const uint64_t len = stg::render_folded(ctx->impl, kind, a, b);
        if (needed) *needed = len + 1;
        if (!buf) return;
        if (cap < len + 1) stg::fail(STG_EINVAL, "buffer too small");
        stg::render_copy(ctx->impl, buf, len);
    });
}

int stg_bundle_load(stg_ctx* ctx, const char* dir, stg_bundle_info* info) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        if (!dir) stg::fail(STG_EINVAL, "null bundle directory");
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        ctx->impl.bundle.reset();
        stg::bundle_load(ctx->impl, dir, info);
    });
}

int stg_bundle_window(stg_ctx* ctx, stg_window* out) {
    return guard([&] {
        if (!ctx->impl.bundle) stg::fail(STG_ESTATE, "no bundle loaded on this context");
        *out = ctx->impl.bundle->w;
    });
}

int stg_device_to_host(stg_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        if (bytes) {
            STG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->impl.stream));
            STG_CUDA(cudaStreamSynchronize(ctx->impl.stream));
        }
    });
}

int stg_aggregate_samples(stg_ctx* ctx, const stg_stream* stream, int64_t drain_interval_ns, int flags,
                          uint64_t* n_windows, uint64_t* n_records) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        if (!stream) stg::fail(STG_EINVAL, "null stream");
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        uint64_t w = 0, r = 0;
        stg::aggregate_samples(ctx->impl, *stream, drain_interval_ns, flags, &w, &r);
        if (n_windows) *n_windows = w;
        if (n_records) *n_records = r;
    });
}

int stg_aggregate_windows(stg_ctx* ctx, int64_t* start_ns, int64_t* end_ns, uint64_t* record_off) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        stg::aggregate_windows(ctx->impl, start_ns, end_ns, record_off);
    });
}

int stg_aggregate_records(stg_ctx* ctx, uint64_t* first_sample, uint64_t* count) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        STG_CUDA(cudaSetDevice(ctx->impl.device));
        stg::aggregate_records(ctx->impl, first_sample, count);
    });
}

int stg_result_folded_text(stg_ctx* ctx, int32_t rank, char* buf, uint64_t cap, uint64_t* needed) {
    return folded_text(ctx, 0, rank, 0, buf, cap, needed);
}

int stg_result_diff_folded(stg_ctx* ctx, int32_t rank_a, int32_t rank_b, char* buf, uint64_t cap,
                           uint64_t* needed) {
    return folded_text(ctx, 1, rank_a, rank_b, buf, cap, needed);
}

}  // extern "C"

static int svg_out(stg_ctx* ctx, int kind, int32_t a, int32_t b, const stg_svg_options* opts, char* buf, uint64_t cap,
                   uint64_t* needed) {
    std::string* text = nullptr;
    int rc = guard([&] {
        std::lock_guard<std::mutex> lk(ctx->impl.mu);
        stg::Result& r = need_result(ctx);
        stg_svg_options o{1200, 16, 0.001, "flame graph"};
        if (opts) o = *opts;
        if (o.width <= 0 || o.row_height <= 0) stg::fail(STG_EINVAL, "svg width and row height must be positive");
        // the text is rendered once per request and handed out by the second call
        uint64_t key = 1469598103934665603ull;
        auto mixin = [&](const void* p, size_t n) {
            for (size_t i = 0; i < n; ++i) key = (key ^ static_cast<const unsigned char*>(p)[i]) * 1099511628211ull;
        };
        mixin(&kind, sizeof kind);
        mixin(&a, sizeof a);
        mixin(&b, sizeof b);
        mixin(&o.width, sizeof o.width);
        mixin(&o.row_height, sizeof o.row_height);
        mixin(&o.min_fraction, sizeof o.min_fraction);
        if (o.title) mixin(o.title, std::strlen(o.title));
        if (r.svg_key != key) {
            r.svg_text = stg::flamegraph_svg(ctx->impl, kind, a, b, o);
            r.svg_key = key;
        }
        text = &r.svg_text;
    });
    if (rc) return rc;
    return copy_out(*text, buf, cap, needed);
}

int stg_result_flamegraph_svg(stg_ctx* ctx, int32_t rank, const stg_svg_options* opts, char* buf, uint64_t cap,
                              uint64_t* needed) {
    return svg_out(ctx, 0, rank, 0, opts, buf, cap, needed);
}

int stg_result_diff_flamegraph_svg(stg_ctx* ctx, int32_t rank_before, int32_t rank_after,
                                   const stg_svg_options* opts, char* buf, uint64_t cap, uint64_t* needed) {
    return svg_out(ctx, 1, rank_before, rank_after, opts, buf, cap, needed);
}
