// stg_runner.inl — host orchestration of one window (included by stg_window.cu).
// Stage order follows build_group_data (bundle.cpp:252-324): collectives first
// (their errors surface first, and the clock offsets feed every other stream),
// then GPU/OS sums, then CPU samples, then the diagnose ladder.
namespace stg {

// Minimal JSON writer (numbers with 17 significant digits: round-trip exact).
struct JsonW {
    std::string s;
    void raw(const char* t) { s += t; }
    void raw(const std::string& t) { s += t; }
    void num(double v) {
        if (!std::isfinite(v)) {
            s += "null";
            return;
        }
        char b[40];
        std::snprintf(b, sizeof b, "%.17g", v);
        s += b;
    }
    void num(int64_t v) { s += std::to_string(v); }
    void num(uint64_t v) { s += std::to_string(v); }
    void num(int v) { s += std::to_string(v); }
    void str(const std::string& t) {
        s += '"';
        for (unsigned char ch : t) {
            switch (ch) {
                case '"': s += "\\\""; break;
                case '\\': s += "\\\\"; break;
                case '\n': s += "\\n"; break;
                case '\t': s += "\\t"; break;
                case '\r': s += "\\r"; break;
                default:
                    if (ch < 0x20) {
                        char b[8];
                        std::snprintf(b, sizeof b, "\\u%04x", ch);
                        s += b;
                    } else {
                        s += char(ch);
                    }
            }
        }
        s += '"';
    }
};

#define LAUNCH(kern, grid, block, ...)                                   \
    do {                                                                 \
        kern<<<(grid), (block), 0, st>>>(__VA_ARGS__);                   \
        STG_CUDA(cudaGetLastError());                                    \
        ++launches;                                                      \
    } while (0)

struct Runner {
    Ctx& c;
    const stg_window& w;
    const stg_config& cfg;
    Result& res;
    cudaStream_t st;
    uint32_t launches = 0, syncs = 0;
    uint64_t h2d = 0, d2h = 0;
    int32_t span = 0;
    // device state shared between stages
    int64_t* d_off = nullptr;
    uint8_t* d_has_off = nullptr;
    double* d_lat = nullptr;
    // samples
    int R = 0;
    uint64_t S = 0;  // dense sequences
    uint64_t L = 0;  // lines
    uint64_t F = 0;  // used names
    uint64_t* d_lkey = nullptr;
    unsigned long long* d_lcount = nullptr;
    uint64_t* d_line_off = nullptr;
    uint64_t* d_seq_off = nullptr;
    uint32_t* d_arena = nullptr;
    uint32_t* d_dense_rep = nullptr;
    uint64_t* d_dn_off = nullptr;
    uint32_t* d_dn = nullptr;
    uint32_t* d_dense_final = nullptr;
    unsigned long long* d_incl = nullptr;
    uint64_t* d_totals = nullptr;
    std::vector<uint64_t> h_n_in;
    std::vector<uint32_t> h_dense_final;
    cudaEvent_t ev[8];
    cudaEvent_t ev_pre = nullptr;   // main-stream point a side-stream stage starts after
    bool gpu_os_done = false;
    uint64_t max_seq_len = 0;

    Runner(Ctx& c_, const stg_window& w_, const stg_config& cfg_, Result& r_)
        : c(c_), w(w_), cfg(cfg_), res(r_), st(c_.stream) {
        for (auto& e : ev) STG_CUDA(cudaEventCreate(&e));
        STG_CUDA(cudaEventCreateWithFlags(&ev_pre, cudaEventDisableTiming));
    }
    ~Runner() {
        for (auto& e : ev) cudaEventDestroy(e);
        cudaEventDestroy(ev_pre);
    }
    // The GPU/OS layer sums (build_group_data bundle.cpp:302-320) do not depend on
    // the sample stream: they run on a side stream (ordered after everything the
    // main stream did before k_sym_agg) while k_sym_agg streams, and their host
    // downloads synchronise only the side stream.
    // The side stream has the highest priority: its few small kernels are
    // scheduled ahead of k_sym_agg's remaining CTAs instead of after them.
    void ensure_side() {
        if (c.side) return;
        int lo = 0, hi = 0;
        STG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        STG_CUDA(cudaStreamCreateWithPriority(&c.side, cudaStreamNonBlocking, hi));
    }
    void side_gpu_os() {
        if (gpu_os_done || side_sharded()) return;  // sharded: main stream, reduced over NCCL after the samples
        ensure_side();
        STG_CUDA(cudaStreamWaitEvent(c.side, ev_pre, 0));
        cudaStream_t keep = st;
        st = c.side;
        try {
            gpu_os();
        } catch (...) {
            st = keep;
            throw;
        }
        st = keep;
        gpu_os_done = true;
    }

    template <class T>
    T* dev(const char* name, size_t n) { return c.buf(name).as<T>(n); }
    template <class T>
    T* up(const char* name, const T* host, size_t n) {
        T* d = dev<T>(name, n);
        if (n) {
            STG_CUDA(cudaMemcpyAsync(d, host, n * sizeof(T), cudaMemcpyHostToDevice, st));
            h2d += n * sizeof(T);
        }
        return d;
    }
    template <class T, class U>
    void down(T* host, const U* d, size_t n) {
        static_assert(sizeof(T) == sizeof(U), "size mismatch");
        if (!n) return;
        STG_CUDA(cudaMemcpyAsync(host, d, n * sizeof(T), cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
        d2h += n * sizeof(T);
        ++syncs;
    }
    template <class T>
    T get1(const T* d) {
        T v;
        down(&v, d, 1);
        return v;
    }
    void zero(void* p, size_t bytes) {
        if (bytes) STG_CUDA(cudaMemsetAsync(p, 0, bytes, st));
    }
    void* temp(size_t bytes) { return c.buf("cub_temp").get(bytes + 16); }

    // ---------------------------------------------------------------- cub
    template <class K, class V>
    void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, uint64_t n, int end_bit = sizeof(K) * 8,
                    int begin_bit = 0) {
        if (!n) return;
        size_t tb = 0;
        STG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, begin_bit, end_bit, st));
        STG_CUDA(cub::DeviceRadixSort::SortPairs(temp(tb), tb, kin, kout, vin, vout, n, begin_bit, end_bit, st));
        ++launches;
    }
    template <class K>
    void sort_keys(const K* kin, K* kout, uint64_t n, int end_bit = sizeof(K) * 8) {
        if (!n) return;
        size_t tb = 0;
        STG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, kin, kout, n, 0, end_bit, st));
        STG_CUDA(cub::DeviceRadixSort::SortKeys(temp(tb), tb, kin, kout, n, 0, end_bit, st));
        ++launches;
    }
    template <class I, class O>
    void excl_sum(const I* in, O* out, uint64_t n) {
        if (!n) return;
        size_t tb = 0;
        STG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, st));
        STG_CUDA(cub::DeviceScan::ExclusiveSum(temp(tb), tb, in, out, n, st));
        ++launches;
    }
    template <class I, class O>
    void incl_sum(const I* in, O* out, uint64_t n) {
        if (!n) return;
        size_t tb = 0;
        STG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, n, st));
        STG_CUDA(cub::DeviceScan::InclusiveSum(temp(tb), tb, in, out, n, st));
        ++launches;
    }
    uint64_t select_flagged(const uint32_t* flags, uint32_t* out, uint64_t n) {
        uint32_t* iota = dev<uint32_t>("sel_iota", n);
        LAUNCH(k_iota, grid_for(n), kThreads, iota, n);
        unsigned long long* nsel = dev<unsigned long long>("sel_n", 1);
        size_t tb = 0;
        STG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, flags, out, nsel, n, st));
        STG_CUDA(cub::DeviceSelect::Flagged(temp(tb), tb, iota, flags, out, nsel, n, st));
        ++launches;
        return get1(nsel);
    }

    // ------------------------------------------------------------ ranks
    const int32_t *cd_rank = nullptr, *cd_group = nullptr;
    const uint8_t* cd_kind = nullptr;
    const int64_t *cd_entry = nullptr, *cd_exit = nullptr;
    int coll_rg[3] = {0, 0, 0};  // min group, max group, max kind
    bool coll_rank_sorted = false;  // event ranks non-decreasing in input order
    void rank_space() {
        int mx = -1, mn = 0;
        for (int32_t i = 0; i < w.n_ranks; ++i) {
            mx = std::max(mx, w.rank_ids[i]);
            mn = std::min(mn, w.rank_ids[i]);
            if (i && w.rank_ids[i] <= w.rank_ids[i - 1])
                fail(STG_EINVAL, "stg_window.rank_ids must be strictly ascending");
        }
        for (int32_t i = 0; i < w.n_group_ranks; ++i) {
            mx = std::max(mx, w.group_ranks[i]);
            mn = std::min(mn, w.group_ranks[i]);
        }
        int* d_mm = dev<int>("mm", 6);  // max rank, min rank, min group, max group, max kind, ranks unsorted
        int init[6] = {mx, mn, INT_MAX, INT_MIN, 0, 0};
        STG_CUDA(cudaMemcpyAsync(d_mm, init, sizeof init, cudaMemcpyHostToDevice, st));
        auto scan = [&](const int32_t* host, uint64_t n, const char* nm) {
            if (!n) return;
            const int32_t* d = up<int32_t>(nm, host, n);
            LAUNCH(k_max_rank, grid_for(n), kThreads, n, d, d_mm, d_mm + 1);
        };
        // collective arrays on the device (uploaded once here when host-resident);
        // their group / kind ranges come back with the rank range
        const uint64_t nc = w.n_coll;
        const bool cdev = w.coll_memory == STG_MEM_DEVICE;
        cd_rank = cdev ? w.coll_rank : (nc ? up<int32_t>("coll_rank", w.coll_rank, nc) : nullptr);
        cd_group = cdev ? w.coll_group : (nc ? up<int32_t>("coll_group", w.coll_group, nc) : nullptr);
        cd_kind = cdev ? w.coll_kind : (nc ? up<uint8_t>("coll_kind", w.coll_kind, nc) : nullptr);
        cd_entry = cdev ? w.coll_entry : (nc ? up<int64_t>("coll_entry", w.coll_entry, nc) : nullptr);
        cd_exit = cdev ? w.coll_exit : (nc ? up<int64_t>("coll_exit", w.coll_exit, nc) : nullptr);
        if (nc) {
            LAUNCH(k_max_rank, grid_for(nc), kThreads, nc, cd_rank, d_mm, d_mm + 1);
            LAUNCH(k_coll_ranges, grid_for(nc), kThreads, nc, cd_group, cd_kind, d_mm + 2, d_mm + 3, d_mm + 4);
            LAUNCH(k_rank_unsorted, grid_for(nc), kThreads, nc, cd_rank, d_mm + 5);
        }
        if (w.side_memory == STG_MEM_DEVICE) {
            if (w.n_gpu) LAUNCH(k_max_rank, grid_for(w.n_gpu), kThreads, w.n_gpu, w.gpu_rank, d_mm, d_mm + 1);
            if (w.n_os) LAUNCH(k_max_rank, grid_for(w.n_os), kThreads, w.n_os, w.os_rank, d_mm, d_mm + 1);
        } else {
            scan(w.gpu_rank, w.n_gpu, "gpu_rank");
            scan(w.os_rank, w.n_os, "os_rank");
        }
        int out[6];
        down(out, d_mm, 6);
        coll_rank_sorted = out[5] == 0;
        coll_rg[0] = out[2];
        coll_rg[1] = out[3];
        coll_rg[2] = out[4];
        if (out[1] < 0) fail(STG_EINVAL, "negative rank ids are not supported");
        if (out[0] >= (1 << 24)) fail(STG_EINVAL, "rank ids must be below 2^24");
        span = out[0] + 1;
    }
    bool coll_sharded() const { return dist() && (w.shard_streams & STG_SHARD_COLL); }
    bool side_sharded() const { return dist() && (w.shard_streams & STG_SHARD_SIDE); }
    // shards of a rank-sharded group: context q owns ranks [sh_lo[q], sh_lo[q+1])
    // and holds sh_n[q] collective events, global event indices from sh_base[q]
    std::vector<int64_t> sh_lo, sh_n, sh_base;
    int r_lo = 0, r_hi = 0;  // this context's ranks, clipped to [0, span)
    void rank_span_agree() {
        if (dist()) {  // every context must index ranks (and collective streams) the same way
            int* d = dev<int>("dx_span", 4);
            int v[4] = {span, coll_rg[1], coll_rg[2], ~coll_rg[0]};  // max of ~g = ~min g
            STG_CUDA(cudaMemcpyAsync(d, v, sizeof v, cudaMemcpyHostToDevice, st));
            nccl(ncclAllReduce(d, d, 4, ncclInt32, ncclMax, comm(), st));
            down(v, d, 4);
            span = v[0];
            if (w.shard_streams & STG_SHARD_COLL) {
                coll_rg[1] = v[1];
                coll_rg[2] = v[2];
                coll_rg[0] = ~v[3];
            }
        }
        res.rank_span = span;
        r_lo = 0;
        r_hi = span;
        if (!(w.shard_streams & (STG_SHARD_COLL | STG_SHARD_SIDE)) || !dist()) return;
        const int W = c.world;
        int64_t* d = dev<int64_t>("dx_shard", 2 * (W + 1));
        int64_t mine[2] = {int64_t(w.shard_rank_lo), int64_t(w.n_coll)};
        STG_CUDA(cudaMemcpyAsync(d + 2 * W, mine, 16, cudaMemcpyHostToDevice, st));
        nccl(ncclAllGather(d + 2 * W, d, 2, ncclInt64, comm(), st));
        std::vector<int64_t> h(2 * W);
        down(h.data(), d, 2 * W);
        sh_lo.assign(W + 1, 0);
        sh_n.assign(W, 0);
        sh_base.assign(W + 1, 0);
        for (int q = 0; q < W; ++q) {
            sh_lo[q] = h[2 * q];
            sh_n[q] = h[2 * q + 1];
            sh_base[q + 1] = sh_base[q] + sh_n[q];
        }
        sh_lo[W] = INT64_MAX;
        for (int q = 1; q < W; ++q)  // identical data on every context: all fail alike
            if (sh_lo[q] <= sh_lo[q - 1])
                fail(STG_EINVAL, "stg_window.shard_rank_lo must increase with the world rank");
        r_lo = int(std::min<int64_t>(std::max<int64_t>(sh_lo[c.wrank], 0), span));
        r_hi = int(std::min<int64_t>(std::max<int64_t>(sh_lo[c.wrank + 1], 0), span));
    }

    // ------------------------------------------------------ collectives
    // one device block for everything the host reads back at the end of stage d
    // (one download): offsets, straggler statistics, error and count words
    uint8_t* cb = nullptr;
    size_t o_ma = 0, o_ml = 0, o_zm = 0, o_fl = 0, o_err = 0, o_cnt = 0, o_has = 0, o_pres = 0, o_hz = 0, o_end = 0;
    uint64_t n_coll_all = 0;  // events stage d runs over (all of them, or the gathered shards)
    void coll_result_init() {
        const uint64_t sp = uint64_t(span);
        o_ma = 8 * sp, o_ml = 16 * sp, o_zm = 24 * sp, o_fl = 32 * sp, o_err = 40 * sp, o_cnt = 40 * sp + 16,
        o_has = 40 * sp + 48, o_pres = 41 * sp + 48, o_hz = 42 * sp + 48, o_end = 43 * sp + 48;
        cb = dev<uint8_t>("c_out", o_end);
        zero(cb, o_end);
        STG_CUDA(cudaMemsetAsync(cb + o_err, 0xff, 16, st));
        d_off = reinterpret_cast<int64_t*>(cb);
        d_has_off = cb + o_has;
        res.n_instances = res.n_windowed = 0;
        res.iteration_times_ms.clear();
        res.offsets.assign(span, 0);
        res.has_offset.assign(span, 0);
        res.lat_present.assign(span, 0);
        res.mean_lat_all.assign(span, 0);
        res.mean_lat_alert.assign(span, 0);
        res.z_mean.assign(span, 0);
        res.flag_count.assign(span, 0);
        res.has_z.assign(span, 0);
        res.have_offsets = false;
    }
    // one download of the result block into the host mirror
    void coll_result_download() {
        const uint64_t sp = uint64_t(span);
        std::vector<uint8_t> h(o_end);
        down(h.data(), cb, o_end);
        std::memcpy(res.offsets.data(), h.data(), 8 * sp);
        std::memcpy(res.mean_lat_all.data(), h.data() + o_ma, 8 * sp);
        std::memcpy(res.mean_lat_alert.data(), h.data() + o_ml, 8 * sp);
        std::memcpy(res.z_mean.data(), h.data() + o_zm, 8 * sp);
        std::memcpy(res.flag_count.data(), h.data() + o_fl, 8 * sp);
        std::memcpy(res.has_offset.data(), h.data() + o_has, sp);
        std::memcpy(res.lat_present.data(), h.data() + o_pres, sp);
        std::memcpy(res.has_z.data(), h.data() + o_hz, sp);
        unsigned long long nd;
        std::memcpy(&nd, h.data() + o_cnt + 16, 8);
        res.have_offsets = nd > 0;
    }
    // column items (regular streams): (stream, chunk of <= kColChunk segments),
    // K[s] events per rank, instance ids from ib[s]
    ColItems col_items(const std::vector<uint32_t>& st_seg_h, const std::vector<uint32_t>& K,
                       const std::vector<uint64_t>& ib) {
        std::vector<uint64_t> off{0}, b;
        std::vector<uint32_t> j0, j1;
        for (size_t s = 0; s + 1 < st_seg_h.size(); ++s)
            for (uint32_t j = st_seg_h[s]; j < st_seg_h[s + 1]; j += kColChunk) {
                j0.push_back(j);
                j1.push_back(std::min<uint32_t>(j + kColChunk, st_seg_h[s + 1]));
                b.push_back(ib[s]);
                off.push_back(off.back() + K[s]);
            }
        ColItems c{};
        c.M = uint32_t(j0.size());
        c.total = off.back();
        if (!c.M) return c;
        c.off = up<uint64_t>("cl_off", off.data(), off.size());
        c.j0 = up<uint32_t>("cl_j0", j0.data(), j0.size());
        c.j1 = up<uint32_t>("cl_j1", j1.data(), j1.size());
        c.ib = up<uint64_t>("cl_ib", b.data(), b.size());
        return c;
    }
    void collectives() {
        const uint64_t sp = uint64_t(span);
        unsigned long long* errs = reinterpret_cast<unsigned long long*>(cb + o_err);
        unsigned long long* cnts = reinterpret_cast<unsigned long long*>(cb + o_cnt);  // n_seg, n_st, n_d, n_w
        const uint64_t n = n_coll_all;
        if (n == 0) return;
        if (n >= 0xffffffffull) fail(STG_EINVAL, "too many collective events");
        zero(cnts + 3, 8);  // n_w
        uint64_t* key = dev<uint64_t>("c_key", n);
        uint64_t* key_s = dev<uint64_t>("c_key_s", n);
        uint32_t* idx = dev<uint32_t>("c_idx", n);
        uint32_t* idx_s = dev<uint32_t>("c_idx_s", n);
        int* d_err = dev<int>("c_err", 1);
        zero(d_err, sizeof(int));
        auto bits_for = [](uint64_t v) { int b = 0; while (b < 64 && (v >> b)) ++b; return b; };
        const int rbits = std::max(1, bits_for(uint64_t(span - 1)));
        const int kbits = std::max(1, bits_for(uint64_t(coll_rg[2])));
        const int gbits = bits_for(uint64_t(int64_t(coll_rg[1]) - coll_rg[0]));
        const uint64_t rmask = (1ull << rbits) - 1;
        LAUNCH(k_coll_keys, grid_for(n), kThreads, n, cd_rank, cd_group, cd_kind, coll_rg[0], kbits, rbits, 0, INT_MAX,
               key, idx, d_err);
        sort_pairs(key, key_s, idx, idx_s, n, gbits + kbits + rbits, coll_rank_sorted ? rbits : 0);
        int64_t* s_entry = dev<int64_t>("c_sentry", n);
        int64_t* s_exit = dev<int64_t>("c_sexit", n);
        uint32_t* seg_flag = dev<uint32_t>("c_segflag", n);
        uint32_t* stream_flag = dev<uint32_t>("c_stflag", n);
        LAUNCH(k_coll_gather, grid_for(n), kThreads, n, key_s, idx_s, cd_entry, cd_exit, rbits, s_entry, s_exit, errs,
               errs + 1, seg_flag, stream_flag);
        // segments (stream, rank) and streams (group, kind), counts on the device
        uint32_t* seg_pos = dev<uint32_t>("c_segpos", n + 1);
        uint32_t* st_pos = dev<uint32_t>("c_stpos", n + 1);
        {
            uint32_t* iota = dev<uint32_t>("sel_iota", n);
            LAUNCH(k_iota, grid_for(n), kThreads, iota, n);
            size_t tb = 0;
            STG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, seg_flag, seg_pos, cnts, n, st));
            STG_CUDA(cub::DeviceSelect::Flagged(temp(tb), tb, iota, seg_flag, seg_pos, cnts, n, st));
            STG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, stream_flag, st_pos, cnts + 1, n, st));
            STG_CUDA(cub::DeviceSelect::Flagged(temp(tb), tb, iota, stream_flag, st_pos, cnts + 1, n, st));
            launches += 2;
        }
        unsigned long long hc[4];  // entry >= exit, order, n_seg, n_st
        {
            std::vector<unsigned long long> h(4);
            STG_CUDA(cudaMemcpyAsync(h.data(), errs, 16, cudaMemcpyDeviceToHost, st));
            STG_CUDA(cudaMemcpyAsync(h.data() + 2, cnts, 16, cudaMemcpyDeviceToHost, st));
            STG_CUDA(cudaStreamSynchronize(st));
            ++syncs;
            for (int q = 0; q < 4; ++q) hc[q] = h[size_t(q)];
        }
        if (hc[0] != ~0ull || hc[1] != ~0ull) {
            if (hc[0] <= hc[1]) fail(STG_EINVAL, "collective event with entry >= exit");
            fail(STG_EINVAL, "collective events not time-ordered within rank");
        }
        const uint64_t n_seg = hc[2], n_st = hc[3];
        {
            const uint32_t nn = uint32_t(n);
            STG_CUDA(cudaMemcpyAsync(seg_pos + n_seg, &nn, 4, cudaMemcpyHostToDevice, st));
        }
        uint32_t* d_st_seg = dev<uint32_t>("c_stseg", n_st + 1);
        uint32_t* d_seg_stream = dev<uint32_t>("c_segstream", n_seg);
        LAUNCH(k_stream_tables, grid_for(n_seg + n_st + 1), kThreads, cnts, seg_pos, st_pos, d_st_seg, d_seg_stream);
        uint32_t* stream_of_pos = dev<uint32_t>("c_streamofpos", n);
        incl_sum(stream_flag, stream_of_pos, n);  // 1-based
        // coarse offsets + counts
        int64_t* coarse = dev<int64_t>("c_coarse", n_seg);
        uint32_t* kmm = dev<uint32_t>("c_kminmax", 2 * n_st);
        uint32_t* kmin = kmm;
        uint32_t* kmax = kmm + n_st;
        LAUNCH(k_coll_streams, unsigned(n_st), kThreads, int(n_st), d_st_seg, seg_pos, s_entry, coarse, kmin, kmax);
        std::vector<uint32_t> h_kmm(2 * n_st);
        down(h_kmm.data(), kmm, 2 * n_st);
        const uint32_t* h_kmin = h_kmm.data();
        const uint32_t* h_kmax = h_kmm.data() + n_st;
        std::vector<uint64_t> k_base(n_st + 1, 0);
        for (uint64_t s = 0; s < n_st; ++s) k_base[s + 1] = k_base[s] + h_kmin[s];
        uint64_t* d_kbase = up<uint64_t>("c_kbase", k_base.data(), n_st + 1);
        uint32_t* first_fail = up<uint32_t>("c_ffail", h_kmin, n_st);
        if (k_base[n_st])
            LAUNCH(k_coll_regular, grid_for(k_base[n_st] * 32), kThreads, int(n_st), d_st_seg, seg_pos, coarse, s_entry,
                   s_exit, kmin, d_kbase, k_base[n_st], w.max_skew_ns, first_fail);
        std::vector<uint32_t> k0(n_st), st_seg_h(n_st + 1);
        STG_CUDA(cudaMemcpyAsync(st_seg_h.data(), d_st_seg, (n_st + 1) * 4, cudaMemcpyDeviceToHost, st));
        down(k0.data(), first_fail, n_st);
        uint32_t* inst_local = dev<uint32_t>("c_instlocal", n);
        uint32_t* d_k0 = first_fail;  // = k0 on the device
        std::vector<int> irregular;
        std::vector<uint32_t> n_inst(n_st);
        for (uint64_t s = 0; s < n_st; ++s) {
            if (k0[s] < h_kmax[s])
                irregular.push_back(int(s));
            else
                n_inst[s] = k0[s];
        }
        const bool col = irregular.empty();  // all regular: column form, no per-event ids
        if (!col) {
            LAUNCH(k_coll_assign_regular, unsigned(std::min<uint64_t>(n_seg, 65535)), 128, int(n_st), d_st_seg,
                   seg_pos, d_seg_stream, uint32_t(n_seg), d_k0, inst_local);
            int* d_irr = up<int>("c_irr", irregular.data(), irregular.size());
            uint32_t* head = dev<uint32_t>("c_head", n_seg);
            uint32_t* d_ninst = dev<uint32_t>("c_ninst", n_st);
            LAUNCH(k_coll_sequential, unsigned(irregular.size()), 1024, d_irr, d_st_seg, seg_pos, coarse, s_entry,
                   s_exit, d_k0, w.max_skew_ns, head, inst_local, d_ninst);
            std::vector<uint32_t> tmp(n_st);
            down(tmp.data(), d_ninst, n_st);
            for (int s : irregular) n_inst[size_t(s)] = tmp[size_t(s)];
        }
        // stream_of_pos is 1-based (inclusive scan): shift the base table
        std::vector<uint64_t> base1(n_st + 1, 0);
        uint64_t I = 0;
        for (uint64_t s = 0; s < n_st; ++s) {
            base1[s + 1] = I;
            I += n_inst[s];
        }
        res.n_instances = I;
        uint64_t* d_ibase = up<uint64_t>("c_ibase", base1.data(), n_st + 1);
        // group membership
        std::vector<uint8_t> member(span, 0);
        unsigned n_group = 0;
        for (int32_t i = 0; i < w.n_group_ranks; ++i)
            if (!member[size_t(w.group_ranks[i])]) {
                member[size_t(w.group_ranks[i])] = 1;
                ++n_group;
            }
        uint8_t* d_member = up<uint8_t>("c_member", member.data(), span);
        uint32_t* inst_of = dev<uint32_t>("c_instof", n);
        unsigned long long* imax = dev<unsigned long long>("c_imax", I);
        unsigned* isize = dev<unsigned>("c_isize", I);
        unsigned* iing = dev<unsigned>("c_iing", I);
        LAUNCH(k_fill_i64, grid_for(I), kThreads, (long long*)imax, I, LLONG_MIN);
        zero(isize, I * sizeof(unsigned));
        zero(iing, I * sizeof(unsigned));
        uint32_t* d_segrank = dev<uint32_t>("c_segrank", n_seg);
        LAUNCH(k_seg_rank, grid_for(n_seg), kThreads, n_seg, seg_pos, key_s, rmask, d_segrank);
        ColItems ci{};
        if (col) {
            std::vector<uint64_t> ib(n_st);
            for (uint64_t s = 0; s < n_st; ++s) ib[s] = base1[s + 1];
            ci = col_items(st_seg_h, k0, ib);
            if (ci.total)
                LAUNCH(k_col_inst, grid_for(ci.total), kThreads, ci, seg_pos, d_segrank, s_exit, d_member, imax, iing);
        } else {
            LAUNCH(k_coll_inst, grid_for(n), kThreads, n, key_s, nullptr, stream_of_pos, d_ibase, inst_local, s_exit,
                   d_member, inst_of, imax, isize, iing, rmask);
        }
        // align_clocks: deltas of complete-instance events, per-rank radix select
        int64_t* dval = dev<int64_t>("c_dval", n);
        long long* d_dmin = dev<long long>("c_dmin", 1);
        zero(d_dmin, 8);
        if (col) {
            if (ci.total)
                LAUNCH(k_col_deltas, grid_for(ci.total), kThreads, ci, seg_pos, s_exit, imax, iing, n_group, dval,
                       d_dmin);
        } else {
            LAUNCH(k_coll_deltas, grid_for(n), kThreads, n, inst_of, s_exit, imax, iing, n_group, dval, d_dmin);
        }
        // per-rank segment lists on the device: segments sorted by their rank
        uint32_t* d_segrank_s = dev<uint32_t>("c_segrank_s", n_seg);
        uint32_t* d_segid = dev<uint32_t>("c_segid", n_seg);
        uint32_t* d_rsegs = dev<uint32_t>("c_rsegs", std::max<uint64_t>(n_seg, 1));
        uint32_t* d_rso = dev<uint32_t>("c_rso", sp + 1);
        LAUNCH(k_iota, grid_for(n_seg), kThreads, d_segid, n_seg);
        sort_pairs(d_segrank, d_segrank_s, d_segid, d_rsegs, n_seg, rbits);
        LAUNCH(k_rank_offsets, grid_for(sp + 1), kThreads, span, d_segrank_s, n_seg, d_rso);
        LAUNCH(k_coll_median_sel, unsigned(std::min<int64_t>(span, 148 * 4)), kMedThreads, int(span), d_rso, d_rsegs, seg_pos,
               dval, d_dmin, d_off, d_has_off, cnts + 2);
        // The clock offsets are all the samples stage needs; the rest of stage d
        // (windowing, lateness, straggler statistics) feeds only the decision
        // ladder, so it runs on the side stream under k_sym_agg (side_coll_tail).
        coll_tail = [=]() {
        // windowed complete instances ordered by max aligned exit
        unsigned long long* aexit = dev<unsigned long long>("c_aexit", I);
        zero(aexit, I * 8);  // int64 0: build_group_data initialises max_exit to 0
        if (col) {
            if (ci.total)
                LAUNCH(k_col_aligned_exit, grid_for(ci.total), kThreads, ci, seg_pos, d_segrank, s_exit, iing, n_group,
                       d_off, aexit);
        } else {
            LAUNCH(k_coll_aligned_exit, grid_for(n), kThreads, n, key_s, inst_of, s_exit, iing, n_group, d_off, aexit,
                   rmask);
        }
        uint64_t* wkey = dev<uint64_t>("c_wkey", I);
        uint64_t* wkey_s = dev<uint64_t>("c_wkey_s", I);
        uint32_t* winst = dev<uint32_t>("c_winst", I);
        uint32_t* winst_s = dev<uint32_t>("c_winst_s", I);
        unsigned long long* nw = cnts + 3;
        LAUNCH(k_coll_window_select, grid_for(I), kThreads, I, iing, n_group, aexit, w.window_start_ns, wkey, winst,
               nw);
        const uint64_t n_w = get1(nw);
        res.n_windowed = n_w;
        sort_pairs(wkey, wkey_s, winst, winst_s, n_w);
        uint32_t* inst_w = dev<uint32_t>("c_instw", I);
        STG_CUDA(cudaMemsetAsync(inst_w, 0xff, I * sizeof(uint32_t), st));
        LAUNCH(k_coll_winv, grid_for(n_w), kThreads, n_w, winst_s, inst_w);
        long long* wmin = dev<long long>("c_wmin", n_w);
        LAUNCH(k_fill_i64, grid_for(n_w), kThreads, wmin, n_w, LLONG_MAX);
        d_lat = dev<double>("lat", sp * n_w);
        LAUNCH(k_fill_f64, grid_for(sp * n_w), kThreads, d_lat, sp * n_w, nan(""));
        if (col) {
            if (ci.total) {
                LAUNCH(k_col_minadj, grid_for(ci.total), kThreads, ci, seg_pos, d_segrank, s_entry, inst_w, d_off, wmin);
                LAUNCH(k_col_lateness, grid_for(ci.total), kThreads, ci, seg_pos, d_segrank, s_entry, inst_w, d_off,
                       wmin, n_w, d_lat);
            }
        } else {
            LAUNCH(k_coll_minadj, grid_for(n), kThreads, n, key_s, inst_of, inst_w, s_entry, d_off, wmin, rmask);
            LAUNCH(k_coll_lateness, grid_for(n), kThreads, n, key_s, inst_of, inst_w, s_entry, d_off, wmin, n_w, d_lat,
                   rmask);
        }
        double* it = dev<double>("c_it", std::max<uint64_t>(n_w, 1));
        if (n_w > 1) LAUNCH(k_coll_itertimes, grid_for(n_w), kThreads, n_w, wkey_s, it);
        // detect_straggler statistics
        if (n_w) {
            double* mu = dev<double>("s_mu", n_w);
            double* sg = dev<double>("s_sg", n_w);
            uint32_t* m = dev<uint32_t>("s_m", n_w);
            double* chain = dev<double>("s_chain", 2 * n_w);
            double* s2 = dev<double>("s_s2", n_w);
            zero(chain, 16 * n_w);
            zero(s2, 8 * n_w);
            strag_chain1(n_w, 0, span, chain);
            LAUNCH(k_strag_mu, grid_for(n_w), kThreads, n_w, chain, mu, m);
            strag_chain2(n_w, 0, span, mu, m, s2);
            LAUNCH(k_strag_sigma, grid_for(n_w), kThreads, n_w, s2, m, sg);
            LAUNCH(k_straggler_rank, grid_for(sp * 32, kStragWarps * 32), kStragWarps * 32, n_w, 0, span, d_lat, cfg.k, mu,
                   sg, m, cb + o_pres, reinterpret_cast<double*>(cb + o_ma), reinterpret_cast<double*>(cb + o_ml),
                   reinterpret_cast<double*>(cb + o_zm), reinterpret_cast<uint64_t*>(cb + o_fl), cb + o_hz);
        }
        // one download for offsets, straggler statistics and counts; one for the iteration times
        if (n_w > 1) {
            res.iteration_times_ms.resize(n_w - 1);
            STG_CUDA(cudaMemcpyAsync(res.iteration_times_ms.data(), it, (n_w - 1) * 8, cudaMemcpyDeviceToHost, st));
            d2h += (n_w - 1) * 8;
        }
        coll_result_download();
        };
    }
    std::function<void()> coll_tail;  // the deferred rest of the replicated stage d
    // run the deferred part of stage d on the side stream (after everything the
    // main stream did before k_sym_agg), or on the main stream when no samples
    // stage gave it a kernel to hide under
    bool side_coll_tail(bool side = true) {
        if (!coll_tail) return false;
        auto f = std::move(coll_tail);
        coll_tail = nullptr;
        if (!side) {
            f();
            return true;
        }
        ensure_side();
        STG_CUDA(cudaStreamWaitEvent(c.side, ev_pre, 0));
        cudaStream_t keep = st;
        st = c.side;
        try {
            f();
        } catch (...) {
            st = keep;
            throw;
        }
        st = keep;
        return true;
    }

    // detect_straggler's per-instance sums (diagnosis.cpp:82-96) over the ranks
    // [r0, r1) in rank order, continuing the chains they are given: a warp per
    // instance for few instances, a thread per instance (coalesced rank rows)
    // for many
    void strag_chain1(uint64_t n_w, int r0, int r1, double* chain) {
        if (n_w >= 4096) LAUNCH(k_strag_chain1_t, grid_for(n_w), kThreads, n_w, r0, r1, d_lat, chain);
        else LAUNCH(k_strag_chain1, grid_for(n_w * 32), kThreads, n_w, r0, r1, d_lat, chain);
    }
    void strag_chain2(uint64_t n_w, int r0, int r1, const double* mu, const uint32_t* m, double* s2) {
        if (n_w >= 4096) LAUNCH(k_strag_chain2_t, grid_for(n_w), kThreads, n_w, r0, r1, d_lat, mu, m, s2);
        else LAUNCH(k_strag_chain2, grid_for(n_w * 32), kThreads, n_w, r0, r1, d_lat, mu, m, s2);
    }

    // ---------------------------------------------- rank-sharded stage d
    // stg_window.shard_streams & STG_SHARD_COLL: every context holds only its
    // ranks' collective events.  coll_local() (may fail; inside agreed()) sorts
    // them into (stream, rank) segments and validates them; coll_exchange()
    // (NCCL, never fails on input) builds the group-wide stream list, proves
    // the regular case with gathered seed candidates, reduces the per-instance
    // partials (max exit, group membership, max aligned exit, min adjusted
    // entry), continues detect_straggler's rank-order sums from context to
    // context (send/recv chain: the single-GPU rounding sequence), and sums the
    // per-rank result blocks.  An irregular stream (missing events, late
    // joiners: the greedy sweep's general case) falls back to gathering every
    // event and running the replicated stage on each context.
    struct CLocal {
        uint64_t n = 0, n_seg = 0, n_st = 0;
        uint64_t* key_s = nullptr;
        int64_t *s_entry = nullptr, *s_exit = nullptr;
        uint32_t *seg_pos = nullptr, *st_pos = nullptr, *stream_of_pos = nullptr, *st_seg = nullptr,
                 *seg_stream = nullptr;
        std::vector<uint64_t> skeys;
        int rbits = 1;
        uint64_t rmask = 1;
    } cl;
    static int bits_for(uint64_t v) {
        int b = 0;
        while (b < 64 && (v >> b)) ++b;
        return b;
    }
    void coll_local() {
        const int W = c.world, P = c.wrank;
        const uint64_t n = w.n_coll;
        cl = CLocal{};
        cl.n = n;
        cl.rbits = std::max(1, bits_for(uint64_t(span - 1)));
        cl.rmask = (1ull << cl.rbits) - 1;
        if (sh_base[W] >= 0xffffffffull) fail(STG_EINVAL, "too many collective events");
        if (n == 0) return;
        unsigned long long* errs = reinterpret_cast<unsigned long long*>(cb + o_err);
        unsigned long long* cnts = reinterpret_cast<unsigned long long*>(cb + o_cnt);
        const int kbits = std::max(1, bits_for(uint64_t(coll_rg[2])));
        const int gbits = bits_for(uint64_t(int64_t(coll_rg[1]) - coll_rg[0]));
        const int rlo = P == 0 ? 0 : int(sh_lo[P]);
        const int rhi = int(std::min<int64_t>(sh_lo[P + 1], INT_MAX));
        uint64_t* key = dev<uint64_t>("c_key", n);
        cl.key_s = dev<uint64_t>("c_key_s", n);
        uint32_t* idx = dev<uint32_t>("c_idx", n);
        uint32_t* idx_s = dev<uint32_t>("c_idx_s", n);
        int* d_err = reinterpret_cast<int*>(cnts + 3);  // n_w word, unused until windowing
        zero(d_err, sizeof(int));
        LAUNCH(k_coll_keys, grid_for(n), kThreads, n, cd_rank, cd_group, cd_kind, coll_rg[0], kbits, cl.rbits, rlo, rhi,
               key, idx, d_err);
        sort_pairs(key, cl.key_s, idx, idx_s, n, gbits + kbits + cl.rbits, coll_rank_sorted ? cl.rbits : 0);
        cl.s_entry = dev<int64_t>("c_sentry", n);
        cl.s_exit = dev<int64_t>("c_sexit", n);
        uint32_t* seg_flag = dev<uint32_t>("c_segflag", n);
        uint32_t* stream_flag = dev<uint32_t>("c_stflag", n);
        LAUNCH(k_coll_gather, grid_for(n), kThreads, n, cl.key_s, idx_s, cd_entry, cd_exit, cl.rbits, cl.s_entry,
               cl.s_exit, errs, errs + 1, seg_flag, stream_flag);
        cl.seg_pos = dev<uint32_t>("c_segpos", n + 1);
        cl.st_pos = dev<uint32_t>("c_stpos", n + 1);
        {
            uint32_t* iota = dev<uint32_t>("sel_iota", n);
            LAUNCH(k_iota, grid_for(n), kThreads, iota, n);
            size_t tb = 0;
            STG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, seg_flag, cl.seg_pos, cnts, n, st));
            STG_CUDA(cub::DeviceSelect::Flagged(temp(tb), tb, iota, seg_flag, cl.seg_pos, cnts, n, st));
            STG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, stream_flag, cl.st_pos, cnts + 1, n, st));
            STG_CUDA(cub::DeviceSelect::Flagged(temp(tb), tb, iota, stream_flag, cl.st_pos, cnts + 1, n, st));
            launches += 2;
        }
        unsigned long long h[6];  // entry >= exit, order, n_seg, n_st, n_d, out-of-shard flag
        STG_CUDA(cudaMemcpyAsync(h, errs, 48, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
        ++syncs;
        if (uint32_t(h[5])) fail(STG_EINVAL, "collective event rank outside the context's shard (shard_rank_lo)");
        if (h[0] != ~0ull || h[1] != ~0ull) {  // the group's first bad event in concatenated order
            fail_rank = int64_t(sh_base[P] + std::min(h[0], h[1]));
            if (h[0] <= h[1]) fail(STG_EINVAL, "collective event with entry >= exit");
            fail(STG_EINVAL, "collective events not time-ordered within rank");
        }
        cl.n_seg = h[2];
        cl.n_st = h[3];
        {
            const uint32_t nn = uint32_t(n);
            STG_CUDA(cudaMemcpyAsync(cl.seg_pos + cl.n_seg, &nn, 4, cudaMemcpyHostToDevice, st));
        }
        cl.st_seg = dev<uint32_t>("c_stseg", cl.n_st + 1);
        cl.seg_stream = dev<uint32_t>("c_segstream", cl.n_seg);
        LAUNCH(k_stream_tables, grid_for(cl.n_seg + cl.n_st + 1), kThreads, cnts, cl.seg_pos, cl.st_pos, cl.st_seg,
               cl.seg_stream);
        cl.stream_of_pos = dev<uint32_t>("c_streamofpos", n);
        incl_sum(stream_flag, cl.stream_of_pos, n);  // 1-based
        uint64_t* skey = dev<uint64_t>("c_skey", cl.n_st);
        LAUNCH(k_stream_keys, grid_for(cl.n_st), kThreads, cnts, cl.st_pos, cl.key_s, cl.rbits, skey);
        cl.skeys.resize(cl.n_st);
        down(cl.skeys.data(), skey, cl.n_st);
    }

    void coll_exchange() {
        const int W = c.world, P = c.wrank;
        if (sh_base[W] == 0) return;
        const uint64_t sp = uint64_t(span), n = cl.n, n_st = cl.n_st, n_seg = cl.n_seg;
        unsigned long long* cnts = reinterpret_cast<unsigned long long*>(cb + o_cnt);
        // 1. the group's (group, kind) streams: sorted union of every context's
        std::vector<uint8_t> mine(n_st * 8);
        if (n_st) std::memcpy(mine.data(), cl.skeys.data(), n_st * 8);
        std::vector<uint64_t> gs;
        for (const auto& b : allgather_bytes(mine))
            for (size_t i = 0; i + 8 <= b.size(); i += 8) {
                uint64_t v;
                std::memcpy(&v, b.data() + i, 8);
                gs.push_back(v);
            }
        std::sort(gs.begin(), gs.end());
        gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
        const uint64_t n_gs = gs.size();
        std::vector<uint32_t> lg(n_st);
        for (uint64_t s = 0; s < n_st; ++s)
            lg[s] = uint32_t(std::lower_bound(gs.begin(), gs.end(), cl.skeys[s]) - gs.begin());
        const uint32_t* d_lg = up<uint32_t>("cs_lg", lg.data(), n_st);
        // 2. per stream: first entry (coarse offsets), per-rank event counts
        long long* minfirst = dev<long long>("cs_minfirst", n_gs);
        uint32_t* kk = dev<uint32_t>("cs_kk", 2 * n_gs);
        LAUNCH(k_fill_i64, grid_for(n_gs), kThreads, minfirst, n_gs, LLONG_MAX);
        zero(kk, 2 * n_gs * 4);
        if (n_st)
            LAUNCH(k_coll_stream_stats, unsigned(n_st), kThreads, int(n_st), cl.st_seg, cl.seg_pos, cl.s_entry, d_lg,
                   uint32_t(n_gs), minfirst, kk);
        nccl(ncclGroupStart());
        nccl(ncclAllReduce(minfirst, minfirst, n_gs, ncclInt64, ncclMin, comm(), st));
        nccl(ncclAllReduce(kk, kk, 2 * n_gs, ncclUint32, ncclMax, comm(), st));
        nccl(ncclGroupEnd());
        int64_t* coarse = dev<int64_t>("c_coarse", n_seg);
        if (n_seg)
            LAUNCH(k_coll_coarse, grid_for(n_seg), kThreads, n_seg, cl.seg_pos, cl.seg_stream, d_lg, cl.s_entry,
                   minfirst, coarse);
        std::vector<uint32_t> h_kk(2 * n_gs), kmax(n_gs), kmin(n_gs);
        down(h_kk.data(), kk, 2 * n_gs);
        for (uint64_t g = 0; g < n_gs; ++g) {
            kmax[g] = h_kk[g];
            kmin[g] = ~h_kk[n_gs + g];
        }
        // 3. regular-case proof: instance k of a stream = every rank's k-th event
        std::vector<uint64_t> k_base(n_gs + 1, 0), lk_base(n_st + 1, 0);
        for (uint64_t g = 0; g < n_gs; ++g) k_base[g + 1] = k_base[g] + kmin[g];
        for (uint64_t s = 0; s < n_st; ++s) lk_base[s + 1] = lk_base[s] + kmin[lg[s]];
        const uint64_t K = k_base[n_gs], nk = lk_base[n_st];
        const uint64_t* d_kbase = up<uint64_t>("cs_kbase", k_base.data(), n_gs + 1);
        const uint64_t* d_lkbase = up<uint64_t>("cs_lkbase", lk_base.data(), n_st + 1);
        long long* cand = dev<long long>("cs_cand", 2 * K);
        long long* cand_all = dev<long long>("cs_cand_all", 2 * K * W);
        uint32_t* ffail = up<uint32_t>("cs_ffail", kmin.data(), n_gs);
        if (K) {
            LAUNCH(k_fill_i64, grid_for(2 * K), kThreads, cand, 2 * K, LLONG_MAX);
            if (nk)
                LAUNCH(k_coll_seed_cand, grid_for(nk * 32), kThreads, int(n_st), cl.st_seg, cl.seg_pos, coarse,
                       cl.s_entry, cl.s_exit, d_lkbase, nk, d_lg, d_kbase, cand);
            nccl(ncclAllGather(cand, cand_all, 2 * K, ncclInt64, comm(), st));
            if (nk)
                LAUNCH(k_coll_regular_sh, grid_for(nk * 32), kThreads, int(n_st), cl.st_seg, cl.seg_pos, coarse,
                       cl.s_entry, cl.s_exit, d_lkbase, nk, d_lg, d_kbase, K, cand_all, W, w.max_skew_ns, ffail);
            nccl(ncclAllReduce(ffail, ffail, n_gs, ncclUint32, ncclMin, comm(), st));
        }
        std::vector<uint32_t> k0(n_gs);
        down(k0.data(), ffail, n_gs);
        for (uint64_t g = 0; g < n_gs; ++g)
            if (k0[g] < kmax[g]) {  // irregular somewhere: the general greedy sweep over all events
                coll_gather_all();
                collectives();
                return;
            }
        // 4. instances (regular: every rank of a stream has k0 events)
        std::vector<uint64_t> ibase(n_gs + 1, 0);
        for (uint64_t g = 0; g < n_gs; ++g) ibase[g + 1] = ibase[g] + k0[g];
        const uint64_t I = ibase[n_gs];
        res.n_instances = I;
        std::vector<uint64_t> base1(n_st + 1, 0);  // stream_of_pos is 1-based
        std::vector<uint32_t> k0l(n_st);
        for (uint64_t s = 0; s < n_st; ++s) {
            base1[s + 1] = ibase[lg[s]];
            k0l[s] = k0[lg[s]];
        }
        // column items over the local segments (every stream is regular here)
        std::vector<uint32_t> st_seg_h(n_st + 1, 0);
        if (n_st) down(st_seg_h.data(), cl.st_seg, n_st + 1);
        std::vector<uint64_t> ib(n_st);
        for (uint64_t s = 0; s < n_st; ++s) ib[s] = base1[s + 1];
        const ColItems ci = col_items(st_seg_h, k0l, ib);
        uint32_t* d_segrank = dev<uint32_t>("c_segrank", n_seg);
        if (n_seg) LAUNCH(k_seg_rank, grid_for(n_seg), kThreads, n_seg, cl.seg_pos, cl.key_s, cl.rmask, d_segrank);
        std::vector<uint8_t> member(span, 0);
        unsigned n_group = 0;
        for (int32_t i = 0; i < w.n_group_ranks; ++i)
            if (!member[size_t(w.group_ranks[i])]) {
                member[size_t(w.group_ranks[i])] = 1;
                ++n_group;
            }
        uint8_t* d_member = up<uint8_t>("c_member", member.data(), span);
        unsigned long long* imax = dev<unsigned long long>("c_imax", I);
        unsigned* iing = dev<unsigned>("c_iing", I);
        LAUNCH(k_fill_i64, grid_for(I), kThreads, (long long*)imax, I, LLONG_MIN);
        zero(iing, I * sizeof(unsigned));
        if (ci.total)
            LAUNCH(k_col_inst, grid_for(ci.total), kThreads, ci, cl.seg_pos, d_segrank, cl.s_exit, d_member, imax,
                   iing);
        nccl(ncclGroupStart());
        nccl(ncclAllReduce(imax, imax, I, ncclInt64, ncclMax, comm(), st));
        nccl(ncclAllReduce(iing, iing, I, ncclUint32, ncclSum, comm(), st));
        nccl(ncclGroupEnd());
        // 5. align_clocks for this context's ranks (medians are per rank)
        if (n) {
            int64_t* dval = dev<int64_t>("c_dval", n);
            long long* d_dmin = dev<long long>("c_dmin", 1);
            zero(d_dmin, 8);
            if (ci.total)
                LAUNCH(k_col_deltas, grid_for(ci.total), kThreads, ci, cl.seg_pos, cl.s_exit, imax, iing, n_group,
                       dval, d_dmin);
            uint32_t* d_segrank_s = dev<uint32_t>("c_segrank_s", n_seg);
            uint32_t* d_segid = dev<uint32_t>("c_segid", n_seg);
            uint32_t* d_rsegs = dev<uint32_t>("c_rsegs", std::max<uint64_t>(n_seg, 1));
            uint32_t* d_rso = dev<uint32_t>("c_rso", sp + 1);
            LAUNCH(k_iota, grid_for(n_seg), kThreads, d_segid, n_seg);
            sort_pairs(d_segrank, d_segrank_s, d_segid, d_rsegs, n_seg, cl.rbits);
            LAUNCH(k_rank_offsets, grid_for(sp + 1), kThreads, span, d_segrank_s, n_seg, d_rso);
            LAUNCH(k_coll_median_sel, unsigned(std::min<int64_t>(span, 148 * 4)), kMedThreads, int(span), d_rso, d_rsegs,
                   cl.seg_pos, dval, d_dmin, d_off, d_has_off, cnts + 2);
        }
        // 6. windowed complete instances, ordered by the max aligned exit
        unsigned long long* aexit = dev<unsigned long long>("c_aexit", I);
        zero(aexit, I * 8);
        if (ci.total)
            LAUNCH(k_col_aligned_exit, grid_for(ci.total), kThreads, ci, cl.seg_pos, d_segrank, cl.s_exit, iing,
                   n_group, d_off, aexit);
        nccl(ncclAllReduce(aexit, aexit, I, ncclInt64, ncclMax, comm(), st));
        uint64_t* wkey = dev<uint64_t>("c_wkey", I);
        uint64_t* wkey_s = dev<uint64_t>("c_wkey_s", I);
        uint32_t* winst = dev<uint32_t>("c_winst", I);
        uint32_t* winst_s = dev<uint32_t>("c_winst_s", I);
        unsigned long long* nw = cnts + 3;
        zero(nw, 8);
        LAUNCH(k_coll_window_select, grid_for(I), kThreads, I, iing, n_group, aexit, w.window_start_ns, wkey, winst,
               nw);
        const uint64_t n_w = get1(nw);
        res.n_windowed = n_w;
        sort_pairs(wkey, wkey_s, winst, winst_s, n_w);
        uint32_t* inst_w = dev<uint32_t>("c_instw", I);
        STG_CUDA(cudaMemsetAsync(inst_w, 0xff, I * sizeof(uint32_t), st));
        LAUNCH(k_coll_winv, grid_for(n_w), kThreads, n_w, winst_s, inst_w);
        long long* wmin = dev<long long>("c_wmin", n_w);
        LAUNCH(k_fill_i64, grid_for(n_w), kThreads, wmin, n_w, LLONG_MAX);
        if (ci.total)
            LAUNCH(k_col_minadj, grid_for(ci.total), kThreads, ci, cl.seg_pos, d_segrank, cl.s_entry, inst_w, d_off,
                   wmin);
        nccl(ncclAllReduce(wmin, wmin, n_w, ncclInt64, ncclMin, comm(), st));
        d_lat = dev<double>("lat", sp * n_w);
        LAUNCH(k_fill_f64, grid_for(sp * n_w), kThreads, d_lat, sp * n_w, nan(""));
        if (ci.total)
            LAUNCH(k_col_lateness, grid_for(ci.total), kThreads, ci, cl.seg_pos, d_segrank, cl.s_entry, inst_w, d_off,
                   wmin, n_w, d_lat);
        double* it = dev<double>("c_it", std::max<uint64_t>(n_w, 1));
        if (n_w > 1) LAUNCH(k_coll_itertimes, grid_for(n_w), kThreads, n_w, wkey_s, it);
        // 7. detect_straggler: per-instance sums in rank order, context after context
        if (n_w) {
            double* chain = dev<double>("s_chain", 2 * n_w);
            double* s2 = dev<double>("s_s2", n_w);
            double* mu = dev<double>("s_mu", n_w);
            double* sg = dev<double>("s_sg", n_w);
            uint32_t* m = dev<uint32_t>("s_m", n_w);
            if (P == 0) zero(chain, 16 * n_w);
            else nccl(ncclRecv(chain, 2 * n_w, ncclFloat64, P - 1, comm(), st));
            strag_chain1(n_w, r_lo, r_hi, chain);
            if (P + 1 < W) nccl(ncclSend(chain, 2 * n_w, ncclFloat64, P + 1, comm(), st));
            nccl(ncclBroadcast(chain, chain, 2 * n_w, ncclFloat64, W - 1, comm(), st));
            LAUNCH(k_strag_mu, grid_for(n_w), kThreads, n_w, chain, mu, m);
            if (P == 0) zero(s2, 8 * n_w);
            else nccl(ncclRecv(s2, n_w, ncclFloat64, P - 1, comm(), st));
            strag_chain2(n_w, r_lo, r_hi, mu, m, s2);
            if (P + 1 < W) nccl(ncclSend(s2, n_w, ncclFloat64, P + 1, comm(), st));
            nccl(ncclBroadcast(s2, s2, n_w, ncclFloat64, W - 1, comm(), st));
            LAUNCH(k_strag_sigma, grid_for(n_w), kThreads, n_w, s2, m, sg);
            if (r_hi > r_lo)
                LAUNCH(k_straggler_rank, grid_for(uint64_t(r_hi - r_lo) * 32, kStragWarps * 32), kStragWarps * 32, n_w,
                       r_lo, r_hi, d_lat, cfg.k, mu, sg, m, cb + o_pres, reinterpret_cast<double*>(cb + o_ma),
                       reinterpret_cast<double*>(cb + o_ml), reinterpret_cast<double*>(cb + o_zm),
                       reinterpret_cast<uint64_t*>(cb + o_fl), cb + o_hz);
        }
        // 8. per-rank blocks (offsets, straggler statistics): each rank's row is
        //    non-zero on its owner only, so sums rebuild the single-context block
        nccl(ncclGroupStart());
        nccl(ncclAllReduce(cb, cb, sp, ncclInt64, ncclSum, comm(), st));
        nccl(ncclAllReduce(cb + o_ma, cb + o_ma, 3 * sp, ncclFloat64, ncclSum, comm(), st));
        nccl(ncclAllReduce(cb + o_fl, cb + o_fl, sp, ncclUint64, ncclSum, comm(), st));
        nccl(ncclAllReduce(cb + o_has, cb + o_has, 3 * sp, ncclUint8, ncclSum, comm(), st));
        nccl(ncclAllReduce(cnts + 2, cnts + 2, 1, ncclUint64, ncclSum, comm(), st));
        nccl(ncclGroupEnd());
        if (n_w > 1) {
            res.iteration_times_ms.resize(n_w - 1);
            STG_CUDA(cudaMemcpyAsync(res.iteration_times_ms.data(), it, (n_w - 1) * 8, cudaMemcpyDeviceToHost, st));
            d2h += (n_w - 1) * 8;
        }
        coll_result_download();
    }

    // Irregular fallback: every context gathers the group's events (its own
    // list concatenated in world-rank order = the group's event order).
    void coll_gather_all() {
        const int W = c.world;
        const uint64_t N = sh_base[W], n = w.n_coll;
        uint64_t mx = 1;
        for (int q = 0; q < W; ++q) mx = std::max<uint64_t>(mx, uint64_t(sh_n[q]));
        auto gather = [&](const void* src, size_t esz, const char* nm_send, const char* nm_pad, const char* nm_out) {
            uint8_t* snd = dev<uint8_t>(nm_send, mx * esz);
            uint8_t* pad = dev<uint8_t>(nm_pad, mx * esz * W);
            uint8_t* out = dev<uint8_t>(nm_out, N * esz);
            if (n) STG_CUDA(cudaMemcpyAsync(snd, src, n * esz, cudaMemcpyDeviceToDevice, st));
            nccl(ncclAllGather(snd, pad, mx * esz, ncclUint8, comm(), st));
            for (int q = 0; q < W; ++q)
                if (sh_n[q])
                    STG_CUDA(cudaMemcpyAsync(out + sh_base[q] * esz, pad + q * mx * esz, sh_n[q] * esz,
                                             cudaMemcpyDeviceToDevice, st));
            return static_cast<const void*>(out);
        };
        cd_rank = static_cast<const int32_t*>(gather(cd_rank, 4, "cg_snd_r", "cg_pad_r", "cg_rank"));
        cd_group = static_cast<const int32_t*>(gather(cd_group, 4, "cg_snd_g", "cg_pad_g", "cg_group"));
        cd_kind = static_cast<const uint8_t*>(gather(cd_kind, 1, "cg_snd_k", "cg_pad_k", "cg_kind"));
        cd_entry = static_cast<const int64_t*>(gather(cd_entry, 8, "cg_snd_e", "cg_pad_e", "cg_entry"));
        cd_exit = static_cast<const int64_t*>(gather(cd_exit, 8, "cg_snd_x", "cg_pad_x", "cg_exit"));
        n_coll_all = N;
        coll_rank_sorted = false;  // the other shards were not checked here
    }

    // ------------------------------------------------------------ gpu/os
    // Per-rank GPU kernel time and OS counter sums (build_group_data
    // bundle.cpp:302-320) in one device block — 8-byte sums / maxima and error
    // flags, then 1-byte presence flags — read back with one download.  With
    // sharded side streams every context fills its own ranks' rows and the
    // block is summed over the group (gpu_os_reduce) before it is read.
    struct SideBlock {
        uint64_t K = 0, C = 1, n8 = 0, n1 = 0;
        size_t o_gs = 0, o_irq = 0, o_sirq = 0, o_p50 = 0, o_p99 = 0, o_mig = 0, o_err = 0;  // in 8-byte words
        size_t o_gp = 0, o_irqp = 0, o_sirqp = 0, o_op = 0;                                 // in bytes after them
        uint8_t* d = nullptr;
        bool gpu = false, os = false;
    } sb;
    void gpu_os() {
        res.gpu.clear();
        res.os.clear();
        const bool shard = side_sharded();
        const bool sdev = w.side_memory == STG_MEM_DEVICE;
        const uint64_t sp = uint64_t(span);
        sb = SideBlock{};
        sb.K = w.n_kernel_names;
        sb.C = std::max<uint32_t>(w.n_counter_names, 1);
        sb.gpu = w.n_gpu || (shard && sb.K);
        sb.os = w.n_os || shard;
        if (!sb.gpu && !sb.os) return;
        size_t q = 0;
        sb.o_gs = q, q += sp * sb.K;
        sb.o_irq = q, q += sp * sb.C;
        sb.o_sirq = q, q += sp * sb.C;
        sb.o_p50 = q, q += sp;
        sb.o_p99 = q, q += sp;
        sb.o_mig = q, q += sp;
        sb.o_err = q, q += 2;
        sb.n8 = q;
        size_t b = 0;
        sb.o_gp = b, b += sp * sb.K;
        sb.o_irqp = b, b += sp * sb.C;
        sb.o_sirqp = b, b += sp * sb.C;
        sb.o_op = b, b += sp;
        sb.n1 = b;
        sb.d = dev<uint8_t>("side_block", sb.n8 * 8 + sb.n1);
        zero(sb.d, sb.n8 * 8 + sb.n1);
        auto w8 = [&](size_t o) { return reinterpret_cast<unsigned long long*>(sb.d) + o; };
        uint8_t* d1 = sb.d + sb.n8 * 8;
        if (w.n_gpu) {
            const uint64_t n = w.n_gpu;
            const int32_t* d_rank = sdev ? w.gpu_rank : static_cast<const int32_t*>(c.buf("gpu_rank").p);
            const uint32_t* d_k = sdev ? w.gpu_kernel : up<uint32_t>("gpu_k", w.gpu_kernel, n);
            const int64_t* d_s = sdev ? w.gpu_start : up<int64_t>("gpu_s", w.gpu_start, n);
            const int64_t* d_d = sdev ? w.gpu_dur : up<int64_t>("gpu_d", w.gpu_dur, n);
            LAUNCH(k_gpu_sums, grid_for(n), kThreads, n, d_rank, d_k, d_s, d_d, d_off, w.window_start_ns,
                   uint32_t(sb.K), w8(sb.o_gs), d1 + sb.o_gp, reinterpret_cast<int*>(w8(sb.o_err)));
        }
        if (w.n_os) {
            const uint64_t n = w.n_os;
            const int32_t* d_rank = sdev ? w.os_rank : static_cast<const int32_t*>(c.buf("os_rank").p);
            const int64_t *ws, *p50, *p99, *mig, *ival, *sval;
            const uint64_t *ioff, *soff;
            const uint32_t *ikey, *skey;
            if (sdev) {
                ws = w.os_window_start;
                p50 = w.os_p50;
                p99 = w.os_p99;
                mig = w.os_migrations;
                ioff = w.os_irq_off;
                ikey = w.os_irq_key;
                ival = w.os_irq_val;
                soff = w.os_sirq_off;
                skey = w.os_sirq_key;
                sval = w.os_sirq_val;
            } else {
                ws = up<int64_t>("os_ws", w.os_window_start, n);
                p50 = up<int64_t>("os_p50", w.os_p50, n);
                p99 = up<int64_t>("os_p99", w.os_p99, n);
                mig = up<int64_t>("os_mig", w.os_migrations, n);
                ioff = up<uint64_t>("os_ioff", w.os_irq_off, n + 1);
                const uint64_t ni = w.os_irq_off[n], ns = w.os_sirq_off[n];
                ikey = up<uint32_t>("os_ikey", w.os_irq_key, ni);
                ival = up<int64_t>("os_ival", w.os_irq_val, ni);
                soff = up<uint64_t>("os_soff", w.os_sirq_off, n + 1);
                skey = up<uint32_t>("os_skey", w.os_sirq_key, ns);
                sval = up<int64_t>("os_sval", w.os_sirq_val, ns);
            }
            LAUNCH(k_os_sums, grid_for(n), kThreads, n, d_rank, ws, p50, p99, mig, ioff, ikey, ival, soff, skey, sval,
                   d_off, w.window_start_ns, uint32_t(w.n_counter_names), w8(sb.o_irq), d1 + sb.o_irqp, w8(sb.o_sirq),
                   d1 + sb.o_sirqp, reinterpret_cast<long long*>(w8(sb.o_p50)),
                   reinterpret_cast<long long*>(w8(sb.o_p99)), w8(sb.o_mig), d1 + sb.o_op,
                   reinterpret_cast<int*>(w8(sb.o_err + 1)));
        }
        if (!shard) gpu_os_collect();
    }
    // sharded side streams: each rank's sums live on the context that owns it
    // (zeros elsewhere; p50 / p99 are maxima of non-negative values), so a sum
    // over the group reproduces the single-context block; the error flags are
    // summed too, so every context sees the same validation result
    void gpu_os_reduce() {
        if (!sb.gpu && !sb.os) return;
        nccl(ncclGroupStart());
        nccl(ncclAllReduce(sb.d, sb.d, sb.n8, ncclInt64, ncclSum, comm(), st));
        nccl(ncclAllReduce(sb.d + sb.n8 * 8, sb.d + sb.n8 * 8, sb.n1, ncclUint8, ncclMax, comm(), st));
        nccl(ncclGroupEnd());
        gpu_os_collect();
    }
    void gpu_os_collect() {
        if (!sb.gpu && !sb.os) return;
        std::vector<uint8_t> h(sb.n8 * 8 + sb.n1);
        down(h.data(), sb.d, h.size());
        const int64_t* h8 = reinterpret_cast<const int64_t*>(h.data());
        const uint8_t* h1 = h.data() + sb.n8 * 8;
        if (int32_t(h8[sb.o_err])) fail(STG_EINVAL, "gpu event kernel index out of range");
        if (int32_t(h8[sb.o_err + 1])) fail(STG_EINVAL, "os counter key index out of range");
        const uint64_t K = sb.K, C = sb.C;
        if (sb.gpu)
            for (int32_t r = 0; r < span; ++r)
                for (uint64_t k = 0; k < K; ++k)
                    if (h1[sb.o_gp + r * K + k]) res.gpu[r][w.kernel_names[k]] += h8[sb.o_gs + r * K + k];
        if (sb.os)
            for (int32_t r = 0; r < span; ++r) {
                if (!h1[sb.o_op + r]) continue;
                OsAcc& a = res.os[r];
                for (uint32_t k = 0; k < w.n_counter_names; ++k) {
                    if (h1[sb.o_irqp + r * C + k]) a.interrupts[w.counter_names[k]] += h8[sb.o_irq + r * C + k];
                    if (h1[sb.o_sirqp + r * C + k]) a.softirqs[w.counter_names[k]] += h8[sb.o_sirq + r * C + k];
                }
                a.p50 = h8[sb.o_p50 + r];
                a.p99 = h8[sb.o_p99 + r];
                a.migrations = h8[sb.o_mig + r];
            }
    }

    // 4 resident CTAs of 8 warps per SM (64 registers); the table staging in
    // shared memory covers up to kMaxSmemBins binaries
    // 4 resident CTAs of 8 warps per SM (64 registers); the table staging in
    // shared memory covers up to kMaxSmemBins binaries
    void launch_sym_agg(const AggParams& p, unsigned grid, bool smem_tabs) {
        if (smem_tabs) {
            k_sym_agg<true, 4, 1, 1><<<grid, kThreads, 0, st>>>(p);
        } else {
            k_sym_agg<false, 4, 1, 1><<<grid, kThreads, 0, st>>>(p);
        }
    }

    // ---------------------------------------------------------- samples
    void samples() {
        R = w.n_ranks;
        res.n_window_ranks = uint32_t(R);
        res.n_gid = 0;
        res.agg_attempts = 0;
        res.pfx_hits = res.pfx_misses = 0;
        res.cpu_rank_ids.clear();
        res.cpu_rank_index.clear();
        res.cpu_totals.clear();
        L = S = F = 0;
        res.n_lines = res.n_seq = res.n_unknown = res.f_used = 0;
        res.unk_final.clear();
        res.unk_labels.clear();
        if (R == 0) return;
        if (R >= (1 << 23)) fail(STG_EINVAL, "too many ranks with CPU samples in one window (limit 2^23)");
        const uint64_t n_s = w.n_samples, n_f = w.n_frames;
        if (w.rank_sample_off[0] != 0 || w.rank_sample_off[R] != n_s)
            fail(STG_EINVAL, "stg_window.rank_sample_off does not cover the samples");
        symtab_refresh_dictionary(c);
        // bulk arrays
        const int64_t *ts;
        const uint64_t *foff, *pc;
        const uint16_t* bin;
        if (w.memory == STG_MEM_DEVICE) {
            if ((reinterpret_cast<uintptr_t>(w.frame_pc) & 31) || (reinterpret_cast<uintptr_t>(w.frame_bin) & 15))
                fail(STG_EINVAL, "device frame_pc must be 32-byte and frame_bin 16-byte aligned");
            ts = w.sample_ts;
            foff = w.sample_frame_off;
            pc = w.frame_pc;
            bin = w.frame_bin;
        } else {
            ts = up<int64_t>("in_ts", w.sample_ts, n_s);
            foff = up<uint64_t>("in_foff", w.sample_frame_off, n_s + 1);
            pc = up<uint64_t>("in_pc", w.frame_pc, n_f);
            bin = up<uint16_t>("in_bin", w.frame_bin, n_f);
        }
        // tables for the window's binaries (missing build id -> every frame unknown)
        std::vector<DevTable> tabs(std::max<int32_t>(w.n_bins, 1));
        for (int32_t b = 0; b < w.n_bins; ++b) {
            DevTable& t = tabs[size_t(b)];
            std::memset(&t, 0, sizeof t);
            auto it = c.table_by_id.find(std::string(reinterpret_cast<const char*>(w.bin_build_ids + 20 * b), 20));
            if (it == c.table_by_id.end()) continue;
            HostTable& h = *c.tables[it->second];
            if (h.n == 0) continue;
            t.e = h.d_e;
            t.bucket = h.d_bucket;
            t.base = h.first_start;
            t.last_start = h.last_start;
            t.shift = h.shift;
            t.nb = h.nb;
            t.n = h.n;
            t.valid = 1;
        }
        DevTable* d_tabs = up<DevTable>("tabs", tabs.data(), tabs.size());
        uint64_t* d_rsoff = up<uint64_t>("rsoff", w.rank_sample_off, R + 1);
        int32_t* d_rids = up<int32_t>("rids", w.rank_ids, R);
        int64_t* d_clk = dev<int64_t>("clk", R);
        LAUNCH(k_clk_of_cpu, grid_for(R), kThreads, R, d_rids, d_off, d_clk);
        std::vector<uint8_t> active(R, 1);
        uint8_t* d_active = up<uint8_t>("active", active.data(), R);
        // per-rank table capacities (remembered across windows)
        std::vector<uint32_t> caps(R);
        for (int r = 0; r < R; ++r) {
            uint64_t nr = w.rank_sample_off[r + 1] - w.rank_sample_off[r];
            uint64_t want = c_cap_hint(r, nr);
            caps[r] = uint32_t(std::max<uint64_t>(64, next_pow2(want)));
        }
        uint32_t unk_cap = uint32_t(std::max<uint64_t>(4096, next_pow2(c_unk_hint())));
        int dev_sms = 148;
        STG_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c.device));
        // everything the host reads after the kernel, in one block (one download):
        // stat[2] | n_in[R] | err_empty[R] | unk_used, unk_ovf, ebin, pad | used[R] | ovf[R] | unsorted[R]
        const size_t so_n = 16 + 16 * size_t(R) + 16 + 12 * size_t(R);
        uint8_t* so = dev<uint8_t>("s_out", so_n);
        unsigned long long* d_stat = reinterpret_cast<unsigned long long*>(so);
        unsigned long long* d_nin = d_stat + 2;
        unsigned long long* d_eempty = d_nin + R;
        unsigned* d_unk_used = reinterpret_cast<unsigned*>(d_eempty + R);
        int* d_unk_ovf = reinterpret_cast<int*>(d_unk_used + 1);
        int* d_ebin = d_unk_ovf + 1;
        unsigned* d_used = reinterpret_cast<unsigned*>(d_ebin + 2);
        int* d_ovf = reinterpret_cast<int*>(d_used + R);
        int* d_uns = d_ovf + R;
        s_unk_used = d_unk_used;
        s_unk_ovf = d_unk_ovf;
        s_ebin = d_ebin;
        std::vector<uint8_t> hso(so_n);
        auto hso_at = [&](const void* dptr) { return hso.data() + (static_cast<const uint8_t*>(dptr) - so); };
        std::vector<uint64_t> tab_off(R);
        // prefix cache: ~4 slots per distinct raw chain of the previous window
        uint32_t pfx_cap = uint32_t(std::min<uint64_t>(1u << 24, std::max<uint64_t>(1u << 16, next_pow2(4 * c.hint_pfx_misses + 1))));
        PfxSlot* pfx = dev<PfxSlot>("pfx", pfx_cap);
        AggSlot* slots = nullptr;
        UnkSlot* unk = nullptr;
        std::vector<int> ovf(R);
        std::vector<unsigned> used(R);
        uint64_t* d_toff = nullptr;
        uint32_t* d_mask = nullptr;
        // bins naming the same build id (verification compares unknown labels by identity)
        std::vector<uint32_t> canon(std::max<int32_t>(w.n_bins, 1));
        for (int32_t b = 0; b < w.n_bins; ++b) {
            canon[size_t(b)] = uint32_t(b);
            for (int32_t a = 0; a < b; ++a)
                if (!std::memcmp(w.bin_build_ids + 20 * a, w.bin_build_ids + 20 * b, 20)) {
                    canon[size_t(b)] = uint32_t(a);
                    break;
                }
        }
        const uint32_t* d_canon = cfg.verify ? up<uint32_t>("bin_canon", canon.data(), canon.size()) : nullptr;
        res.verify_retries = 0;
        res.verified = 0;
        // Verification passes: pass 0 is the normal run; after a detected
        // collision the stage re-runs with re-keyed fingerprints and without the
        // prefix cache (stg_config.verify).
        for (int pass = 0;; ++pass) {
        AggParams p{};
        for (int attempt = 0;; ++attempt) {
            uint64_t tot = 0;
            for (int r = 0; r < R; ++r) {
                tab_off[r] = tot;
                tot += caps[r];
            }
            if (tot >= (1ull << 32)) fail(STG_ENOMEM, "aggregation tables exceed 2^32 slots");
            slots = dev<AggSlot>("slots", tot);
            zero(slots, tot * sizeof(AggSlot));
            d_toff = up<uint64_t>("toff", tab_off.data(), R);
            std::vector<uint32_t> masks(R);
            for (int r = 0; r < R; ++r) masks[r] = caps[r] - 1;
            d_mask = up<uint32_t>("tmask", masks.data(), R);
            unk = dev<UnkSlot>("unk", unk_cap);
            zero(unk, size_t(unk_cap) * sizeof(UnkSlot));
            zero(so, so_n);
            STG_CUDA(cudaMemsetAsync(d_eempty, 0xff, R * 8, st));
            p = AggParams{};
            p.ts = ts;
            p.foff = foff;
            p.pc = pc;
            p.bin = bin;
            p.rank_soff = d_rsoff;
            p.rank_clk = d_clk;
            p.active = d_active;
            p.R = R;
            p.ws = w.window_start_ns;
            p.tabs = d_tabs;
            p.n_bins = uint32_t(w.n_bins);
            p.mode = cfg.lookup_mode;
            p.slots = slots;
            p.tab_off = d_toff;
            p.tab_mask = d_mask;
            p.tab_used = d_used;
            p.tab_overflow = d_ovf;
            p.unk = UnkSet{unk, unk_cap - 1, unk_cap / 2, d_unk_used, d_unk_ovf};
            p.n_in = d_nin;
            p.unsorted = d_uns;
            p.err_empty = d_eempty;
            p.err_bin = d_ebin;
            p.n_samples = n_s;
            p.n_frames = n_f;
            p.pfx = pfx;
            p.pfx_mask = pfx_cap - 1;
            p.stat = d_stat;
            p.salt = pass ? 0x9e3779b97f4a7c15ull * uint64_t(pass) + 0x2545f4914f6cdd1dull : 0;
            p.use_pfx = pass == 0;
            p.weak_pfx = cfg.debug_weak_prefix_key != 0;
            zero(pfx, size_t(pfx_cap) * sizeof(PfxSlot));
            // 4 resident CTAs of 8 warps per SM (64 registers), 16 waves' worth of
            // CTAs: each warp owns a contiguous batch range, so the CTAs in flight
            // cover a narrow slice of the rank-major samples — few ranks' hash
            // tables are hot in L2 at a time (C2: 17.5 -> 16.2 ms against 4 waves,
            // profiles/r2e_grid_sweep.md) and the last wave's tail is short
            const uint64_t need = ((n_s + 31) / 32 + (kThreads / 32) - 1) / (kThreads / 32);
            unsigned grid = unsigned(dev_sms) * 64;
            if (need < grid) grid = unsigned(std::max<uint64_t>(need, 1));
            cudaEventRecord(ev[2], st);
            if (attempt == 0 && pass == 0) cudaEventRecord(ev_pre, st);
            launch_sym_agg(p, grid, w.n_bins <= kMaxSmemBins);
            STG_CUDA(cudaGetLastError());
            ++launches;
            cudaEventRecord(ev[3], st);
            if (attempt == 0) {  // host + side-stream work while the kernel streams
                side_gpu_os();
                side_coll_tail();
            }
            res.agg_attempts = attempt + 1;
            down(hso.data(), so, so_n);
            mark("s:k_sym_agg");
            std::memcpy(ovf.data(), hso_at(d_ovf), R * 4);
            std::memcpy(used.data(), hso_at(d_used), R * 4);
            bool any = false;
            for (int r = 0; r < R; ++r)
                if (ovf[r] || used[r] > (caps[r] >> 1)) {  // probe cap hit, or past the 50 % load limit
                    caps[r] = caps[r] >= (1u << 30) ? caps[r] : caps[r] * 4;
                    any = true;
                }
            bool unk_over = *reinterpret_cast<const int*>(hso_at(d_unk_ovf)) != 0;
            if (unk_over) unk_cap = unk_cap >= (1u << 30) ? unk_cap : unk_cap * 4;
            if (!any && !unk_over) break;
            if (attempt > 6) fail(STG_ENOMEM, "aggregation tables kept overflowing");
        }
        c_set_hints(used, *reinterpret_cast<const unsigned*>(hso_at(d_unk_used)));
        {
            unsigned long long hm[2];
            std::memcpy(hm, hso_at(d_stat), 16);
            res.pfx_hits = hm[0];
            res.pfx_misses = hm[1];
            if (pass == 0) c.hint_pfx_misses = uint32_t(std::min<unsigned long long>(hm[1], 1u << 22));
        }
        if (*reinterpret_cast<const int*>(hso_at(d_ebin))) fail(STG_EINVAL, "frame binary index out of range");
        h_n_in.resize(R);
        std::memcpy(h_n_in.data(), hso_at(d_nin), R * 8);
        // validation in aggregate_samples order (samples.cpp:32-58), ranks ascending;
        // a rank whose in-window samples all have empty stacks has no aggregated
        // sample but still fails like the reference
        std::vector<unsigned long long> eempty(R), ereg(R, ~0ull);
        std::memcpy(eempty.data(), hso_at(d_eempty), R * 8);
        std::vector<int> uns(R);
        std::memcpy(uns.data(), hso_at(d_uns), R * 4);
        std::vector<int> flagged;
        for (int r = 0; r < R; ++r)
            if (uns[r] && h_n_in[r]) flagged.push_back(r);
        if (!flagged.empty()) {
            int* d_fl = up<int>("regr_r", flagged.data(), flagged.size());
            unsigned long long* d_o = dev<unsigned long long>("regr_o", flagged.size());
            LAUNCH(k_regress_exact, grid_for(flagged.size(), 64), 64, int(flagged.size()), d_fl, d_rsoff, ts, d_clk,
                   w.window_start_ns, d_o);
            std::vector<unsigned long long> o(flagged.size());
            down(o.data(), d_o, flagged.size());
            for (size_t i = 0; i < flagged.size(); ++i) ereg[size_t(flagged[i])] = o[i];
        }
        int64_t drain = w.window_end_ns - w.window_start_ns + 2 * w.max_skew_ns;
        for (int r = 0; r < R; ++r) {
            if (!h_n_in[r] && eempty[r] == ~0ull) continue;
            fail_rank = w.rank_ids[r];
            if (drain <= 0) fail(STG_EINVAL, "drain interval must be positive");
            if (eempty[r] != ~0ull || ereg[r] != ~0ull) {
                if (eempty[r] <= ereg[r]) fail(STG_EINVAL, "empty sample stack");
                fail(STG_EINVAL, "aggregate_samples: timestamps regressed");
            }
        }
        fail_rank = -1;
        res.cpu_rank_ids.clear();
        res.cpu_rank_index.clear();
        res.cpu_totals.clear();
        for (int r = 0; r < R; ++r)
            if (h_n_in[r]) {
                res.cpu_rank_ids.push_back(w.rank_ids[r]);
                res.cpu_rank_index.push_back(uint32_t(r));
                res.cpu_totals.push_back(h_n_in[r]);
            }
        d_totals = up<uint64_t>("totals", h_n_in.data(), R);
        mark("s:validate");
        if (cfg.verify && !verify_aggregation(p, d_canon, tab_off[R - 1] + caps[R - 1])) {
            if (pass >= 2) fail(STG_ECUDA, "verification failed after re-keyed retries");
            ++res.verify_retries;
            continue;
        }
        fold(slots, tab_off, caps, unk, unk_cap, d_rsoff, foff, pc, bin, d_tabs, d_canon);
        if (cfg.verify && fold_bad) {
            if (pass >= 2) fail(STG_ECUDA, "verification failed after re-keyed retries");
            ++res.verify_retries;
            continue;
        }
        res.verified = cfg.verify ? 1 : 0;
        break;
        }
    }

    // stg_config.verify, stage a+b: every in-window sample against its slot's
    // representative, slot counts recounted (k_sym_verify, k_count_check).
    bool verify_aggregation(const AggParams& p, const uint32_t* d_canon, uint64_t n_slots) {
        unsigned* vc = dev<unsigned>("v_count", n_slots);
        zero(vc, n_slots * 4);
        unsigned long long* bad = dev<unsigned long long>("v_bad", 1);
        zero(bad, 8);
        LAUNCH(k_sym_verify, 148 * 8, kThreads, p, d_canon, vc, bad);
        LAUNCH(k_count_check, grid_for(n_slots), kThreads, n_slots, p.slots, vc, bad);
        const bool ok = get1(bad) == 0;
        mark("s:verify");
        return ok;
    }
    bool fold_bad = false;
    unsigned* s_unk_used = nullptr;  // inside the samples stage's output block
    int *s_unk_ovf = nullptr, *s_ebin = nullptr;
    int64_t fail_rank = -1;  // rank (or group event index) whose validation failed (distributed error agreement)

    // table-capacity hints kept on the context between windows
    uint64_t c_cap_hint(int r, uint64_t nr) {
        const auto& v = c.hint_rank_used;
        uint64_t base = std::min<uint64_t>(2 * nr + 2, 1u << 15);
        if (size_t(r) < v.size() && v[size_t(r)]) base = std::min<uint64_t>(2 * nr + 2, uint64_t(v[size_t(r)]) * 2 + 64);
        return base;
    }
    uint64_t c_unk_hint() {
        return c.hint_rank_used.empty() ? 4096 : uint64_t(c.hint_unk_used) * 2 + 1024;
    }
    void c_set_hints(const std::vector<unsigned>& used, unsigned unk_used) {
        c.hint_rank_used.assign(used.begin(), used.end());
        c.hint_unk_used = unk_used;
    }

    // Unknown labels (symfile.cpp:159-163) merged into the sorted name space.
    // Real name i moves to i + #{non-name labels < name i}; a label that equals a
    // real name shares its rank, so folding merges them exactly like strings.
    uint64_t n_pos = 0;
    void merge_labels(uint32_t NU, const std::vector<uint32_t>& hs, const std::vector<uint32_t>& hb,
                      const std::vector<uint64_t>& hp, uint32_t unk_cap) {
        const auto& dict = c.dict;
        res.dict = &c.dict;
        res.unk_final.clear();
        if (c.label_pos_version != c.dict_version || c.label_pos.size() > (1u << 20)) {  // per dictionary, bounded
            c.label_pos.clear();
            c.label_pos_version = c.dict_version;
        }
        res.unk_labels.clear();
        std::vector<std::pair<std::string, uint32_t>> labels(NU);
        for (uint32_t i = 0; i < NU; ++i) labels[i] = {unknown_label(w.bin_build_ids + 20 * hb[i], hp[i]), hs[i]};
        std::sort(labels.begin(), labels.end());
        std::vector<uint32_t> unk_final_by_slot(unk_cap, 0), pos_sorted;
        uint64_t ne_before = 0;
        uint64_t last_final = 0;
        for (uint32_t i = 0; i < NU; ++i) {
            const std::string& lab = labels[i].first;
            if (i > 0 && lab == labels[i - 1].first) {  // same label from two slots
                unk_final_by_slot[labels[i].second] = uint32_t(last_final);
                continue;
            }
            uint64_t pos;
            bool eq;
            auto ci = c.label_pos.find(lab);
            if (ci != c.label_pos.end()) {
                pos = ci->second.first;
                eq = ci->second.second;
            } else {
                pos = uint64_t(dict.lower_bound(lab));
                eq = pos < dict.size() && dict[pos] == lab;
                c.label_pos.emplace(lab, std::make_pair(pos, eq));
            }
            uint64_t fr = pos + ne_before;
            unk_final_by_slot[labels[i].second] = uint32_t(fr);
            last_final = fr;
            if (!eq) {
                pos_sorted.push_back(uint32_t(pos));
                res.unk_final.push_back(fr);
                res.unk_labels.push_back(lab);
                ++ne_before;
            }
        }
        up<uint32_t>("u_final", unk_final_by_slot.data(), unk_cap);
        n_pos = pos_sorted.size();
        uint32_t zero32 = 0;
        up<uint32_t>("u_pos", n_pos ? pos_sorted.data() : &zero32, std::max<uint64_t>(n_pos, 1));
    }

    // -------------------------------------------------------------- fold
    void fold(AggSlot* slots, const std::vector<uint64_t>& tab_off, const std::vector<uint32_t>& caps, UnkSlot* unk,
              uint32_t unk_cap, const uint64_t* d_rsoff, const uint64_t* foff, const uint64_t* pc,
              const uint16_t* bin, const DevTable* d_tabs, const uint32_t* d_canon) {
        cudaEventRecord(ev[4], st);
        fold_bad = false;
        uint64_t tot = 0;
        uint32_t maxcap = 0;
        for (int r = 0; r < R; ++r) {
            tot += caps[r];
            maxcap = std::max(maxcap, caps[r]);
        }
        uint64_t* d_toff = static_cast<uint64_t*>(c.buf("toff").p);
        uint32_t* d_mask = static_cast<uint32_t*>(c.buf("tmask").p);
        uint64_t Lmax = 0;
        for (int r = 0; r < R; ++r) Lmax += std::min<uint64_t>(caps[r], w.rank_sample_off[r + 1] - w.rank_sample_off[r]);
        Lmax = std::max<uint64_t>(Lmax, 1);
        uint32_t* l_rank = dev<uint32_t>("l_rank", Lmax);
        uint64_t* l_hi = dev<uint64_t>("l_hi", Lmax);
        uint64_t* l_lo = dev<uint64_t>("l_lo", Lmax);
        uint32_t* l_cnt32 = dev<uint32_t>("l_cnt32", Lmax);
        uint64_t* l_rep = dev<uint64_t>("l_rep", Lmax);
        unsigned long long* nl = dev<unsigned long long>("nl", 1);
        zero(nl, 8);
        dim3 g(std::max(1u, std::min(64u, (maxcap + kThreads - 1) / kThreads)), unsigned(R));
        k_compact_lines<<<g, kThreads, 0, st>>>(R, d_toff, d_mask, slots, d_rsoff, l_rank, l_hi, l_lo, l_cnt32,
                                                 l_rep, nl);
        STG_CUDA(cudaGetLastError());
        ++launches;
        L = get1(nl);
        res.n_lines = L;
        mark("f:compact");
        if (L == 0) return;
        // global dedupe -> sequence ids.  The table is sized from the previous
        // window's distinct count (lines repeat the same stacks across ranks), with a
        // retry at 2 slots per line if it fills up.
        unsigned long long* dstat = dev<unsigned long long>("seq_stat", 3);
        uint32_t* l_gid = dev<uint32_t>("l_gid", L);
        uint64_t* seq_rep = dev<uint64_t>("seq_rep", L);
        const uint64_t scap_full = next_pow2(2 * L);
        uint64_t scap = std::min<uint64_t>(scap_full, next_pow2(std::max<uint64_t>(4 * uint64_t(c.hint_gid) + 1024, 1u << 16)));
        uint32_t G = 0;
        uint64_t A = 0;
        for (;;) {
            SeqSlot* sslots = dev<SeqSlot>("sslots", scap);
            LAUNCH(k_fill_gid, grid_for(scap), kThreads, sslots, scap);  // clears the slots, gid = unpublished
            zero(dstat, 24);
            LAUNCH(k_seq_dedupe, grid_for(L), kThreads, L, l_hi, l_lo, l_rep, sslots, scap - 1, dstat, l_gid, seq_rep,
                   foff);
            unsigned long long hs3[3];
            down(hs3, dstat, 3);
            G = uint32_t(hs3[0]);
            A = hs3[1];
            max_seq_len = hs3[2];
            if (!(hs3[0] >> 32)) break;
            if (scap >= scap_full) fail(STG_ENOMEM, "sequence table overflow");
            scap = scap_full;
        }
        c.hint_gid = G;
        res.n_gid = G;
        mark("f:dedupe");
        // materialize
        uint64_t* seq_len = dev<uint64_t>("seq_len", G + 1);
        LAUNCH(k_seq_len64, grid_for(G), kThreads, G, seq_rep, foff, seq_len);
        zero(seq_len + G, 8);
        d_seq_off = dev<uint64_t>("seq_off", G + 1);
        excl_sum(seq_len, d_seq_off, uint64_t(G) + 1);
        d_arena = dev<uint32_t>("arena", std::max<uint64_t>(A, 1));
        unsigned* d_unk_used = s_unk_used;
        int* d_unk_ovf = s_unk_ovf;
        int* d_ebin = s_ebin;
        UnkSet us{unk, unk_cap - 1, unk_cap - 1, d_unk_used, d_unk_ovf};
        LAUNCH(k_seq_materialize, grid_for(uint64_t(G) * 32), kThreads, G, seq_rep, d_seq_off, foff, pc, bin, d_tabs,
               uint32_t(w.n_bins), cfg.lookup_mode, us, d_ebin, d_arena);
        if (cfg.verify) {  // every line's stack against its sequence representative
            unsigned long long* bad = dev<unsigned long long>("v_bad", 1);
            zero(bad, 8);
            LAUNCH(k_line_verify, 148 * 8, kThreads, L, l_rep, l_gid, seq_rep, foff, pc, bin, d_tabs, uint32_t(w.n_bins),
                   cfg.lookup_mode, us, d_ebin, d_canon, bad);
            if (get1(bad)) {
                fold_bad = true;
                return;
            }
            mark("f:verify");
        }
        // unknown labels -> merged name space
        ulonglong2* u_rec = dev<ulonglong2>("u_rec", unk_cap);
        unsigned* nu = dev<unsigned>("nu", 1);
        zero(nu, 4);
        LAUNCH(k_unk_compact, grid_for(unk_cap), kThreads, unk_cap, unk, u_rec, nu);
        uint32_t NU = get1(nu);
        res.n_unknown = NU;
        std::vector<ulonglong2> ur(NU);
        down(ur.data(), u_rec, NU);
        std::vector<uint32_t> hs(NU), hb(NU);
        std::vector<uint64_t> hp(NU);
        for (uint32_t k = 0; k < NU; ++k) {
            hp[k] = ur[k].x;
            hs[k] = uint32_t(ur[k].y);
            hb[k] = uint32_t(ur[k].y >> 32);
        }
        merge_labels(NU, hs, hb, hp, unk_cap);
        mark("f:labels");
        LAUNCH(k_remap, grid_for(A), kThreads, A, d_arena, static_cast<const uint32_t*>(c.buf("u_final").p),
               static_cast<const uint32_t*>(c.buf("u_pos").p), uint32_t(n_pos));
        uint64_t NF = c.dict.size() + res.unk_labels.size();
        res.n_names = NF;
        // lexicographic order of the sequences
        uint32_t* seq_rank = dev<uint32_t>("seq_rank", G);
        {
            const uint64_t maxlen = max_seq_len;  // from the dedupe stats
            int p_log = 1;
            while ((uint64_t(1) << p_log) < maxlen) ++p_log;
            const uint64_t n0 = uint64_t(G) << p_log;
            if (n0 <= (1ull << 27)) {
                // prefix doubling (k_pd_*): log2(P) radix sorts of shrinking pair-key arrays
                uint32_t* cur = dev<uint32_t>("pd_cur", n0);
                LAUNCH(k_pd_init, grid_for(n0), kThreads, n0, uint32_t(p_log), d_seq_off, d_arena, cur);
                uint64_t* key = dev<uint64_t>("pd_key", n0 / 2);
                uint64_t* key_s = dev<uint64_t>("pd_key_s", n0 / 2);
                uint32_t* idx = dev<uint32_t>("pd_idx", n0 / 2);
                uint32_t* idx_s = dev<uint32_t>("pd_idx_s", n0 / 2);
                uint32_t* flg = dev<uint32_t>("pd_flag", n0 / 2);
                uint32_t* rnk = dev<uint32_t>("pd_rank", n0 / 2);
                uint64_t n = n0;
                uint64_t vmax = NF + 1;  // level-0 values: name + 1, sentinel 0
                for (int lvl = 1; lvl <= p_log; ++lvl) {
                    n /= 2;
                    int vb = 1;
                    while ((uint64_t(1) << vb) <= vmax) ++vb;
                    LAUNCH(k_pd_pairs, grid_for(n), kThreads, n, cur, vb, key, idx);
                    sort_pairs(key, key_s, idx, idx_s, n, 2 * vb);
                    LAUNCH(k_pd_flags, grid_for(n), kThreads, n, key_s, flg);
                    incl_sum(flg, rnk, n);
                    LAUNCH(k_pd_scatter, grid_for(n), kThreads, n, idx_s, rnk, cur);
                    vmax = n;  // dense ranks 1..(distinct blocks) <= n
                }
                S = get1(rnk + (G - 1));
                res.n_seq = S;
                d_dense_rep = dev<uint32_t>("dense_rep", S);
                LAUNCH(k_pd_final, grid_for(G), kThreads, G, cur, seq_rank, d_dense_rep);
            } else {  // very deep stacks: comparator merge sort
                uint32_t* gids = dev<uint32_t>("gids", G);
                LAUNCH(k_iota, grid_for(G), kThreads, gids, G);
                SeqLess less{d_arena, d_seq_off};
                size_t tb = 0;
                STG_CUDA(cub::DeviceMergeSort::SortKeys(nullptr, tb, gids, int64_t(G), less, st));
                STG_CUDA(cub::DeviceMergeSort::SortKeys(temp(tb), tb, gids, int64_t(G), less, st));
                ++launches;
                uint32_t* fl = dev<uint32_t>("sq_flag", G);
                uint32_t* scn = dev<uint32_t>("sq_scan", G);
                LAUNCH(k_seq_rankflags, grid_for(G), kThreads, G, gids, less, fl);
                incl_sum(fl, scn, G);
                S = get1(scn + G - 1);
                res.n_seq = S;
                d_dense_rep = dev<uint32_t>("dense_rep", S);
                LAUNCH(k_seq_rankset, grid_for(G), kThreads, G, gids, scn, seq_rank, d_dense_rep);
            }
            mark("f:seqsort");
            uint64_t* lkey = dev<uint64_t>("lkey", L);
            LAUNCH(k_line_keys, grid_for(L), kThreads, L, l_rank, l_gid, seq_rank, lkey);
            d_lkey = dev<uint64_t>("lkey_s", L);
            unsigned long long* lc64 = dev<unsigned long long>("lc64", L);
            LAUNCH(k_u32_to_u64, grid_for(L), kThreads, L, l_cnt32, lc64);
            d_lcount = dev<unsigned long long>("lcount_s", L);
            int rb = 1;  // line key = rank << 32 | sequence rank: sort only the bits in use
            while ((uint64_t(1) << rb) < uint64_t(R)) ++rb;
            sort_pairs(lkey, d_lkey, lc64, d_lcount, L, 32 + rb);
            if (S < G) {  // identical name sequences from distinct keys: merge lines
                uint64_t* uk = dev<uint64_t>("rbk_k", L);
                unsigned long long* uv = dev<unsigned long long>("rbk_v", L);
                unsigned long long* nr = dev<unsigned long long>("rbk_n", 1);
                size_t tb2 = 0;
                STG_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, tb2, d_lkey, uk, d_lcount, uv, nr, cub::Sum(), L, st));
                STG_CUDA(cub::DeviceReduce::ReduceByKey(temp(tb2), tb2, d_lkey, uk, d_lcount, uv, nr, cub::Sum(), L, st));
                ++launches;
                L = get1(nr);
                res.n_lines = L;
                STG_CUDA(cudaMemcpyAsync(d_lkey, uk, L * 8, cudaMemcpyDeviceToDevice, st));
                STG_CUDA(cudaMemcpyAsync(d_lcount, uv, L * 8, cudaMemcpyDeviceToDevice, st));
            }
        }
        d_line_off = dev<uint64_t>("line_off", R + 1);
        LAUNCH(k_line_bounds, grid_for(R + 1), kThreads, R, d_lkey, L, d_line_off);
        mark("f:linesort");
        cudaEventRecord(ev[5], st);
        // ---- stage c: distinct names per sequence, used-name space, inclusive counts
        uint64_t* dcnt = dev<uint64_t>("dn_cnt", S + 1);
        uint32_t* dcnt32 = dev<uint32_t>("dn_cnt32", S + 1);
        LAUNCH(k_seq_distinct<false>, grid_for(S * 32), kThreads, uint32_t(S), d_dense_rep, d_seq_off, d_arena, dcnt32,
               nullptr, nullptr);
        zero(dcnt32 + S, 4);
        LAUNCH(k_u32_to_u64, grid_for(S + 1), kThreads, S + 1, dcnt32, (unsigned long long*)dcnt);
        d_dn_off = dev<uint64_t>("dn_off", S + 1);
        excl_sum(dcnt, d_dn_off, S + 1);
        // distinct names per sequence <= its length: size by the arena, count stays on the device
        const uint64_t ND = A;
        res.f_nd_bound = std::max<uint64_t>(ND, 1);
        d_dn = dev<uint32_t>("dn", std::max<uint64_t>(ND, 1));
        LAUNCH(k_seq_distinct<true>, grid_for(S * 32), kThreads, uint32_t(S), d_dense_rep, d_seq_off, d_arena, nullptr,
               d_dn_off, d_dn);
        uint32_t* used = dev<uint32_t>("used", NF + 1);
        zero(used, (NF + 1) * 4);
        LAUNCH(k_mark_used, grid_for(ND), kThreads, d_dn_off + S, d_dn, used);
        uint32_t* used_scan = dev<uint32_t>("used_scan", NF + 1);
        excl_sum(used, used_scan, NF + 1);
        F = get1(used_scan + NF);
        res.f_used = F;
        mark("f:names");
        d_dense_final = dev<uint32_t>("dense_final", F);
        LAUNCH(k_dense_final, grid_for(NF), kThreads, NF, used, used_scan, d_dense_final);
        LAUNCH(k_dense_names, grid_for(ND), kThreads, d_dn_off + S, d_dn, used_scan);
        cudaEventRecord(ev[6], st);
    }

    // Inclusive counts per (window rank, name), incl[r * F + f]; only
    // the waterline needs them, so they are computed on request.
    bool incl_done = false;
    void inclusive_counts() {
        if (incl_done) return;
        incl_done = true;
        const uint64_t cells = uint64_t(R) * F;
        if (cells > (1ull << 33)) fail(STG_ENOMEM, "rank x name matrix too large");
        d_incl = dev<unsigned long long>("incl", std::max<uint64_t>(cells, 1));
        zero(d_incl, cells * 8);
        if (!F || !L) return;
        const uint32_t Rp = uint32_t((R + 3) & ~3);
        const uint64_t cm = uint64_t(S) * Rp;
        const uint64_t* nd_ptr = d_dn_off + S;
        if (cm * 4 <= (4ull << 30)) {
            uint32_t* C = dev<uint32_t>("incl_c", cm);
            zero(C, cm * 4);
            LAUNCH(k_lines_to_mat, grid_for(L), kThreads, L, d_lkey, d_lcount, Rp, C);
            const uint64_t nd = get1(nd_ptr);
            uint32_t* pf = dev<uint32_t>("incl_pf", std::max<uint64_t>(nd, 1));
            uint32_t* ps = dev<uint32_t>("incl_ps", std::max<uint64_t>(nd, 1));
            uint32_t* col_f = dev<uint32_t>("incl_colf", std::max<uint64_t>(nd, 1));
            uint32_t* col_s = dev<uint32_t>("incl_cols", std::max<uint64_t>(nd, 1));
            LAUNCH(k_name_pairs, grid_for(uint64_t(S) * 32), kThreads, uint32_t(S), d_dn_off, d_dn, pf, ps);
            int fb = 1;
            while (fb < 32 && (uint64_t(1) << fb) < F) ++fb;
            sort_pairs(pf, col_f, ps, col_s, nd, fb);
            // column slices per warp: enough warps to fill the GPU, <= 512 entries each
            const uint32_t seg = uint32_t(std::max<uint64_t>(8, std::min<uint64_t>(512, nd / (148ull * 32) + 1)));
            LAUNCH(k_incl_spmm, grid_for((nd + seg - 1) / seg * 32), kThreads, nd_ptr, col_f, col_s, C, uint32_t(R), Rp,
                   F, seg, d_incl);
        } else {
            LAUNCH(k_incl_lines, grid_for(L * 32), kThreads, L, d_lkey, d_lcount, d_dn_off, d_dn, F, d_incl);
        }
        mark("w:incl");
    }

    // ------------------------------------------------------- diagnose
    std::string dense_name(uint32_t f) {
        if (h_dense_final.size() != F) {
            h_dense_final.resize(F);
            down(h_dense_final.data(), d_dense_final, F);
        }
        return res.name_of(h_dense_final[f]);
    }
    // names of a few dense indices: gathered on the device unless the whole
    // dense -> name map is already on the host (or most of it is wanted)
    std::vector<std::string> dense_names(const std::vector<uint32_t>& fs) {
        std::vector<std::string> out;
        out.reserve(fs.size());
        if (h_dense_final.size() == F || fs.size() * 64 >= F) {
            for (uint32_t f : fs) out.push_back(dense_name(f));
            return out;
        }
        if (fs.empty()) return out;
        const uint32_t* q = up<uint32_t>("dn_q", fs.data(), fs.size());
        uint32_t* g = dev<uint32_t>("dn_g", fs.size());
        LAUNCH(k_gather_u32, grid_for(fs.size()), kThreads, uint64_t(fs.size()), q, d_dense_final, g);
        std::vector<uint32_t> h(fs.size());
        down(h.data(), g, h.size());
        for (uint32_t k : h) out.push_back(res.name_of(k));
        return out;
    }
    int cpu_index(int rank) const {
        auto it = std::lower_bound(res.cpu_rank_ids.begin(), res.cpu_rank_ids.end(), rank);
        if (it == res.cpu_rank_ids.end() || *it != rank) return -1;
        return int(res.cpu_rank_index[size_t(it - res.cpu_rank_ids.begin())]);
    }
    std::vector<std::string> seq_names(uint32_t s) {
        uint32_t g;
        down(&g, d_dense_rep + s, 1);
        uint64_t o[2];
        down(o, d_seq_off + g, 2);
        std::vector<uint32_t> keys(o[1] - o[0]);
        down(keys.data(), d_arena + o[0], keys.size());
        std::vector<std::string> out;
        for (uint32_t k : keys) out.push_back(res.name_of(k));
        return out;
    }
    // hottest path over lines [a, b) of the sorted line list (or over sequences)
    std::vector<std::string> hottest(uint64_t a, uint64_t b, uint32_t f, bool merged) {
        unsigned long long* best = dev<unsigned long long>("hot_best", 2);
        unsigned long long init[2] = {0, ~0ull};
        STG_CUDA(cudaMemcpyAsync(best, init, 16, cudaMemcpyHostToDevice, st));
        if (merged) {
            auto sc = static_cast<unsigned long long*>(c.buf("seq_counts").p);
            for (int pass = 0; pass < 2; ++pass)
                LAUNCH(k_hottest, grid_for(uint64_t(S) * 32), kThreads, S, nullptr, sc, 1, d_dn_off, d_dn, f, pass, best);
        } else {
            for (int pass = 0; pass < 2; ++pass)
                LAUNCH(k_hottest, grid_for((b - a) * 32), kThreads, b - a, d_lkey + a, d_lcount + a, 0, d_dn_off, d_dn, f, pass,
                       best);
        }
        // one download for the winner's whole name sequence
        const uint32_t cap = uint32_t(std::max<uint64_t>(max_seq_len, 1));
        uint32_t* pk = dev<uint32_t>("hot_pack", size_t(cap) + 2);
        LAUNCH(k_hot_pack, 1, 256, best, merged ? nullptr : d_lkey + a, merged ? 1 : 0, d_dense_rep, d_seq_off, d_arena,
               cap, pk);
        std::vector<uint32_t> hp(size_t(cap) + 2);
        down(hp.data(), pk, hp.size());
        if (!hp[0]) return {};
        if (hp[1] > cap) {  // longer than any sequence seen at the sort: fall back
            unsigned long long hb[2];
            down(hb, best, 2);
            uint32_t s;
            if (merged)
                s = uint32_t(hb[1]);
            else {
                uint64_t k;
                down(&k, d_lkey + a + hb[1], 1);
                s = uint32_t(k);
            }
            return seq_names(s);
        }
        std::vector<std::string> out;
        out.reserve(hp[1]);
        for (uint32_t k = 0; k < hp[1]; ++k) out.push_back(res.name_of(hp[2 + k]));
        return out;
    }
    // Exact inclusive fractions over lines [a, a+n) (or over all sequences when
    // merged): returns (dense name, fraction) in name order.
    using Fracs = std::vector<std::pair<uint32_t, double>>;
    Fracs exact_fractions(uint64_t a, uint64_t n, uint64_t total, bool merged, const uint64_t* dn_off = nullptr,
                          const uint32_t* dn = nullptr, const unsigned long long* counts = nullptr) {
        return std::move(exact_fractions2(a, n, total, 0, 0, 0, merged, dn_off, dn, counts, nullptr)[0]);
    }
    // Two line ranges in one pass (the straggler and the reference rank): one
    // pair sort with the side in the key, all the running sums in one launch.
    std::array<Fracs, 2> exact_fractions2(uint64_t a0, uint64_t n0, uint64_t t0, uint64_t a1, uint64_t n1, uint64_t t1,
                                          bool merged, const uint64_t* dn_off = nullptr, const uint32_t* dn = nullptr,
                                          const unsigned long long* counts = nullptr, const uint8_t* want = nullptr) {
        std::array<Fracs, 2> out;
        if (t0 == 0) n0 = 0;
        if (t1 == 0) n1 = 0;
        const uint64_t n = n0 + n1;
        if (n == 0) return out;
        const uint64_t* d_dn_off = dn_off ? dn_off : this->d_dn_off;
        const uint32_t* d_dn = dn ? dn : this->d_dn;
        const uint64_t* lk0 = merged ? nullptr : d_lkey + a0;
        const uint64_t* lk1 = merged ? nullptr : d_lkey + a1;
        const unsigned long long* cnt0 =
            counts ? counts : (merged ? static_cast<unsigned long long*>(c.buf("seq_counts").p) : d_lcount + a0);
        const unsigned long long* cnt1 = merged ? cnt0 : d_lcount + a1;
        int LB = 1;
        while ((uint64_t(1) << LB) < std::max(n0, n1)) ++LB;
        uint64_t* pc = dev<uint64_t>("xf_cnt", n + 1);
        LAUNCH(k_pair_count, grid_for(n * 32), kThreads, n, n0, lk0, lk1, d_dn_off, d_dn, want, pc);
        zero(pc + n, 8);
        uint64_t* po = dev<uint64_t>("xf_off", n + 1);
        excl_sum(pc, po, n + 1);
        uint64_t np = get1(po + n);
        if (!np) return out;
        uint64_t* keys = dev<uint64_t>("xf_keys", np);
        uint64_t* keys_s = dev<uint64_t>("xf_keys_s", np);
        double* vals = dev<double>("xf_vals", np);
        double* vals_s = dev<double>("xf_vals_s", np);
        // names of the window's own dictionary are dense (< F); caller-given
        // global keys may use all 31 bits
        int NB = 31;
        if (!dn) {
            NB = 1;
            while (NB < 31 && (uint64_t(1) << NB) < F) ++NB;
        }
        LAUNCH(k_pair_emit, grid_for(n * 32), kThreads, n, n0, lk0, lk1, cnt0, cnt1, t0, t1, d_dn_off, d_dn, want, po, LB,
               NB, keys, vals);
        // pairs are emitted in line order and the radix sort is stable, so
        // sorting the (side, name) bits alone keeps each name's lines in order
        sort_pairs(keys, keys_s, vals, vals_s, np, LB + NB + 1, LB);
        uint32_t* flag = dev<uint32_t>("xf_flag", np);
        LAUNCH(k_pair_segflags, grid_for(np), kThreads, np, keys_s, LB, flag);
        uint32_t* seg = dev<uint32_t>("xf_seg", np);
        uint64_t nseg = select_flagged(flag, seg, np);
        uint32_t* of = dev<uint32_t>("xf_of", nseg);
        double* ov = dev<double>("xf_ov", nseg);
        LAUNCH(k_pair_segsum, grid_for(nseg * 32, kSegWarps * 32), kSegWarps * 32, nseg, seg, np, keys_s, LB, NB, vals_s,
               of, ov);
        std::vector<uint32_t> hf(nseg);
        std::vector<double> hv(nseg);
        down(hf.data(), of, nseg);
        down(hv.data(), ov, nseg);
        for (uint64_t i = 0; i < nseg; ++i) out[hf[i] >> 31].push_back({hf[i] & 0x7fffffffu, hv[i]});
        return out;
    }
    static double mean_of(const std::vector<double>& v) {
        double s = 0.0;
        for (double x : v) s += x;
        return s / double(v.size());
    }
    static double pstd(const std::vector<double>& v, double mu) {
        double a = 0.0;
        for (double x : v) a += (x - mu) * (x - mu);
        return std::sqrt(a / double(v.size()));
    }
    static double median_of(std::vector<double> v) {
        std::sort(v.begin(), v.end());
        size_t n = v.size();
        return n % 2 ? v[n / 2] : (v[n / 2 - 1] + v[n / 2]) / 2.0;
    }

    // ============================================================ distributed
    bool dist() const { return c.comm != nullptr && c.world > 1; }
    ncclComm_t comm() const { return static_cast<ncclComm_t>(c.comm); }
    void nccl(ncclResult_t r) {
        if (r != ncclSuccess) fail(STG_ECUDA, std::string("NCCL: ") + ncclGetErrorString(r));
    }
    std::vector<uint8_t> bcast_bytes(std::vector<uint8_t> buf, int root) {
        uint64_t* dn = dev<uint64_t>("dx_n", 1);
        uint64_t n = buf.size();
        STG_CUDA(cudaMemcpyAsync(dn, &n, 8, cudaMemcpyHostToDevice, st));
        nccl(ncclBroadcast(dn, dn, 1, ncclUint64, root, comm(), st));
        n = get1(dn);
        buf.resize(n);
        if (!n) return buf;
        uint8_t* d = dev<uint8_t>("dx_b", n);
        if (c.wrank == root) STG_CUDA(cudaMemcpyAsync(d, buf.data(), n, cudaMemcpyHostToDevice, st));
        nccl(ncclBroadcast(d, d, n, ncclUint8, root, comm(), st));
        down(buf.data(), d, n);
        return buf;
    }
    std::vector<std::vector<uint8_t>> allgather_bytes(const std::vector<uint8_t>& mine) {
        const int W = c.world;
        uint64_t* dn = dev<uint64_t>("dx_sizes", W + 1);
        uint64_t n = mine.size();
        STG_CUDA(cudaMemcpyAsync(dn + W, &n, 8, cudaMemcpyHostToDevice, st));
        nccl(ncclAllGather(dn + W, dn, 1, ncclUint64, comm(), st));
        std::vector<uint64_t> sz(W);
        down(sz.data(), dn, W);
        uint64_t mx = 1;
        for (uint64_t v : sz) mx = std::max(mx, v);
        uint8_t* dm = dev<uint8_t>("dx_mine", mx);
        if (n) STG_CUDA(cudaMemcpyAsync(dm, mine.data(), n, cudaMemcpyHostToDevice, st));
        uint8_t* da = dev<uint8_t>("dx_all", mx * W);
        nccl(ncclAllGather(dm, da, mx, ncclUint8, comm(), st));
        std::vector<uint8_t> all(mx * W);
        down(all.data(), da, mx * W);
        std::vector<std::vector<uint8_t>> out(W);
        for (int r = 0; r < W; ++r) out[r].assign(all.begin() + r * mx, all.begin() + r * mx + sz[r]);
        return out;
    }
    template <class T>
    static void put(std::vector<uint8_t>& b, T v) {
        const uint8_t* p = reinterpret_cast<const uint8_t*>(&v);
        b.insert(b.end(), p, p + sizeof(T));
    }
    static void put_str(std::vector<uint8_t>& b, const std::string& s) {
        put<uint32_t>(b, uint32_t(s.size()));
        b.insert(b.end(), s.begin(), s.end());
    }
    template <class T>
    static T get(const uint8_t*& p) {
        T v;
        std::memcpy(&v, p, sizeof(T));
        p += sizeof(T);
        return v;
    }
    static std::string get_str(const uint8_t*& p) {
        uint32_t n = get<uint32_t>(p);
        std::string s(reinterpret_cast<const char*>(p), n);
        p += n;
        return s;
    }

    // Global name keys: the byte-wise sorted union of the (identical) symbol
    // dictionary and every context's unknown labels, so keys compare like the
    // strings on every GPU.
    struct GNames {
        std::vector<uint64_t> lab_final;
        std::vector<std::string> lab;
        std::vector<uint32_t> pos;
        std::vector<uint64_t> loc_final;   // local label finals (sorted)
        std::vector<uint32_t> loc_global;  // their global keys
    } gn;
    bool gn_ready = false;
    void global_names() {
        if (gn_ready) return;
        if (c.dict_hash_version != c.dict_version) {  // once per dictionary
            uint64_t hv = 1469598103934665603ull;
            for (size_t i = 0; i < c.dict.size(); ++i) {
                for (unsigned char ch : c.dict[i]) hv = (hv ^ ch) * 1099511628211ull;
                hv = (hv ^ 0xff) * 1099511628211ull;
            }
            c.dict_hash = hv;
            c.dict_hash_version = c.dict_version;
        }
        const uint64_t h = c.dict_hash;
        if (c.dict_agreed_version != c.dict_version) {
        unsigned long long* dh = dev<unsigned long long>("dx_h", 2);
        unsigned long long hh[2] = {h, h};
        STG_CUDA(cudaMemcpyAsync(dh, hh, 16, cudaMemcpyHostToDevice, st));
        nccl(ncclAllReduce(dh, dh, 1, ncclUint64, ncclMin, comm(), st));
        nccl(ncclAllReduce(dh + 1, dh + 1, 1, ncclUint64, ncclMax, comm(), st));
        down(hh, dh, 2);
        if (hh[0] != hh[1]) fail(STG_EINVAL, "distributed contexts hold different symbol tables");
        c.dict_agreed_version = c.dict_version;
        }
        mark("g:agree");
        // each label travels with its dictionary position (known from
        // merge_labels: final = pos + index among labels), so the merge needs
        // no search in the dictionary
        std::vector<uint8_t> mine;
        put<uint32_t>(mine, uint32_t(res.unk_labels.size()));
        for (size_t k = 0; k < res.unk_labels.size(); ++k) {
            put<uint32_t>(mine, uint32_t(res.unk_final[k] - k));
            put_str(mine, res.unk_labels[k]);
        }
        std::vector<std::pair<std::string, uint32_t>> all;
        auto gathered = allgather_bytes(mine);
        mark("g:allgather");
        for (const auto& b : gathered) {  // each context's labels arrive sorted: merge
            const uint8_t* p = b.data();
            uint32_t n = b.empty() ? 0 : get<uint32_t>(p);
            const size_t o = all.size();
            for (uint32_t i = 0; i < n; ++i) {
                uint32_t pos = get<uint32_t>(p);
                all.emplace_back(get_str(p), pos);
            }
            if (!std::is_sorted(all.begin() + o, all.end())) std::sort(all.begin() + o, all.end());
            std::inplace_merge(all.begin(), all.begin() + o, all.end());
        }
        all.erase(std::unique(all.begin(), all.end(),
                              [](const auto& a, const auto& b) { return a.first == b.first; }),
                  all.end());
        uint64_t ne_before = 0;
        for (const auto& [lab, pos] : all) {
            gn.lab.push_back(lab);
            gn.lab_final.push_back(uint64_t(pos) + ne_before);
            gn.pos.push_back(pos);
            ++ne_before;
        }
        for (size_t k = 0; k < res.unk_labels.size(); ++k) {
            size_t gi = size_t(std::lower_bound(gn.lab.begin(), gn.lab.end(), res.unk_labels[k]) - gn.lab.begin());
            gn.loc_final.push_back(res.unk_final[k]);
            gn.loc_global.push_back(uint32_t(gn.lab_final[gi]));
        }
        gn_ready = true;
        mark("g:merge");
    }
    uint32_t to_global(uint32_t f) const {
        auto it = std::lower_bound(gn.loc_final.begin(), gn.loc_final.end(), uint64_t(f));
        if (it != gn.loc_final.end() && *it == f) return gn.loc_global[size_t(it - gn.loc_final.begin())];
        uint64_t i = f - uint64_t(it - gn.loc_final.begin());
        return uint32_t(i + uint64_t(std::upper_bound(gn.pos.begin(), gn.pos.end(), uint32_t(i)) - gn.pos.begin()));
    }
    std::string gname(uint32_t g) const {
        auto it = std::lower_bound(gn.lab_final.begin(), gn.lab_final.end(), uint64_t(g));
        if (it != gn.lab_final.end() && *it == g) return gn.lab[size_t(it - gn.lab_final.begin())];
        return std::string(c.dict[g - uint64_t(it - gn.lab_final.begin())]);
    }
    // owner context of each rank's CPU profile (-1: none anywhere)
    std::vector<int32_t> cpu_owner;
    void cpu_owners() {
        std::vector<int32_t> own(span, 0);
        for (int32_t r : res.cpu_rank_ids) own[size_t(r)] = c.wrank + 1;
        int32_t* d = up<int32_t>("dx_owner", own.data(), span);
        nccl(ncclAllReduce(d, d, span, ncclInt32, ncclMax, comm(), st));
        down(own.data(), d, span);
        cpu_owner.resize(span);
        for (int32_t r = 0; r < span; ++r) cpu_owner[r] = own[r] - 1;
    }
    // this context's exact fractions of CPU rank `rank` as (global key, value),
    // plus the dense index of each key for local follow-ups
    // dense name of a global key on this context (-1: not used here): the
    // inverse of to_global, checked by the round trip
    int64_t dense_of_global(uint32_t g) const {
        uint64_t fin;
        auto it = std::lower_bound(gn.lab_final.begin(), gn.lab_final.end(), uint64_t(g));
        if (it != gn.lab_final.end() && *it == g) {  // a label: find it among this context's labels
            const std::string& lab = gn.lab[size_t(it - gn.lab_final.begin())];
            auto lt = std::lower_bound(res.unk_labels.begin(), res.unk_labels.end(), lab);
            if (lt == res.unk_labels.end() || *lt != lab) return -1;
            fin = res.unk_final[size_t(lt - res.unk_labels.begin())];
        } else {  // a dictionary name: i, shifted by this context's labels sorting before it
            const uint64_t i = g - uint64_t(it - gn.lab_final.begin());
            uint64_t lo = 0, hi = res.unk_final.size();  // labels whose dictionary position <= i
            while (lo < hi) {
                const uint64_t mid = (lo + hi) / 2;
                if (res.unk_final[mid] - mid <= i) lo = mid + 1; else hi = mid;
            }
            fin = i + lo;
        }
        auto dt = std::lower_bound(h_dense_final.begin(), h_dense_final.end(), uint32_t(fin));
        if (dt == h_dense_final.end() || *dt != fin) return -1;
        const uint32_t f = uint32_t(dt - h_dense_final.begin());
        return to_global(h_dense_final[f]) == g ? int64_t(f) : -1;
    }
    std::vector<std::string> bcast_path(std::vector<std::string> path, int root) {
        std::vector<uint8_t> b;
        if (c.wrank == root)
            for (const auto& n : path) put_str(b, n);
        b = bcast_bytes(std::move(b), root);
        std::vector<std::string> out;
        for (const uint8_t* p = b.data(); p < b.data() + b.size();) out.push_back(get_str(p));
        return out;
    }

    // Temporal route across GPUs: every context contributes its merged
    // (all local ranks) stacks in global keys; each GPU re-merges the union,
    // sorts it in std::map order and sums fractions in that order.
    struct MergedSeqs {
        uint64_t n = 0, total = 0;
        uint32_t* arena = nullptr;
        uint64_t* off = nullptr;
        unsigned long long* cnt = nullptr;
        uint64_t* dn_off = nullptr;
        uint32_t* dn = nullptr;
    };
    MergedSeqs merged_union() {
        MergedSeqs m;
        std::vector<uint8_t> mine;
        uint64_t T = 0;
        for (uint64_t t : res.cpu_totals) T += t;
        put<uint64_t>(mine, T);
        if (S > 0 && L > 0) {
            auto sc = dev<unsigned long long>("seq_counts", S);
            zero(sc, S * 8);
            LAUNCH(k_seq_counts, grid_for(L), kThreads, L, d_lkey, d_lcount, sc);
            std::vector<unsigned long long> hsc(S);
            down(hsc.data(), sc, S);
            std::vector<uint32_t> drep(S);
            down(drep.data(), d_dense_rep, S);
            std::vector<uint64_t> soff(res.n_gid + 1);
            down(soff.data(), d_seq_off, res.n_gid + 1);
            std::vector<uint32_t> ar(soff[res.n_gid]);
            down(ar.data(), d_arena, ar.size());
            for (uint64_t s = 0; s < S; ++s) {
                if (!hsc[s]) continue;
                uint32_t g = drep[s];
                put<uint64_t>(mine, hsc[s]);
                put<uint32_t>(mine, uint32_t(soff[g + 1] - soff[g]));
                for (uint64_t k = soff[g]; k < soff[g + 1]; ++k) put<uint32_t>(mine, to_global(ar[k]));
            }
        }
        std::vector<uint32_t> keys;
        std::vector<uint64_t> off{0};
        std::vector<unsigned long long> cnt;
        for (const auto& b : allgather_bytes(mine)) {
            const uint8_t* p = b.data();
            const uint8_t* e = b.data() + b.size();
            m.total += get<uint64_t>(p);
            while (p < e) {
                cnt.push_back(get<uint64_t>(p));
                uint32_t n = get<uint32_t>(p);
                for (uint32_t k = 0; k < n; ++k) keys.push_back(get<uint32_t>(p));
                off.push_back(keys.size());
            }
        }
        const uint64_t n = cnt.size();
        if (!n) return m;
        uint32_t* d_keys = up<uint32_t>("mg_keys", keys.data(), keys.size());
        uint64_t* d_off = up<uint64_t>("mg_off", off.data(), off.size());
        unsigned long long* d_cnt = up<unsigned long long>("mg_cnt", cnt.data(), n);
        uint32_t* idx = dev<uint32_t>("mg_idx", n);
        LAUNCH(k_iota, grid_for(n), kThreads, idx, n);
        SeqLess less{d_keys, d_off};
        size_t tb = 0;
        STG_CUDA(cub::DeviceMergeSort::SortKeys(nullptr, tb, idx, int64_t(n), less, st));
        STG_CUDA(cub::DeviceMergeSort::SortKeys(temp(tb), tb, idx, int64_t(n), less, st));
        ++launches;
        uint32_t* flg = dev<uint32_t>("mg_flag", n);
        uint32_t* scn = dev<uint32_t>("mg_scan", n);
        LAUNCH(k_seq_rankflags, grid_for(n), kThreads, uint32_t(n), idx, less, flg);
        incl_sum(flg, scn, n);
        const uint64_t nm = get1(scn + n - 1);
        uint32_t* rep = dev<uint32_t>("mg_rep", nm);
        uint32_t* rank_of = dev<uint32_t>("mg_rankof", n);
        LAUNCH(k_seq_rankset, grid_for(n), kThreads, uint32_t(n), idx, scn, rank_of, rep);
        unsigned long long* mc = dev<unsigned long long>("mg_mcnt", nm);
        zero(mc, nm * 8);
        LAUNCH(k_scatter_add, grid_for(n), kThreads, n, rank_of, d_cnt, mc);
        // distinct names per merged stack (dense_rep = representative index)
        uint32_t* c32 = dev<uint32_t>("mg_c32", nm + 1);
        LAUNCH(k_seq_distinct<false>, grid_for(nm * 32), kThreads, uint32_t(nm), rep, d_off, d_keys, c32, nullptr, nullptr);
        zero(c32 + nm, 4);
        uint64_t* c64 = dev<uint64_t>("mg_c64", nm + 1);
        LAUNCH(k_u32_to_u64, grid_for(nm + 1), kThreads, nm + 1, c32, (unsigned long long*)c64);
        uint64_t* dn_off = dev<uint64_t>("mg_dnoff", nm + 1);
        excl_sum(c64, dn_off, nm + 1);
        const uint64_t nd = get1(dn_off + nm);
        uint32_t* dn = dev<uint32_t>("mg_dn", nd);
        LAUNCH(k_seq_distinct<true>, grid_for(nm * 32), kThreads, uint32_t(nm), rep, d_off, d_keys, nullptr, dn_off, dn);
        m.n = nm;
        m.arena = d_keys;
        m.off = d_off;
        m.cnt = mc;
        m.dn_off = dn_off;
        m.dn = dn;
        merged_rep = rep;
        return m;
    }
    uint32_t* merged_rep = nullptr;
    std::vector<std::string> merged_path(const MergedSeqs& m, uint32_t key) {
        unsigned long long* best = dev<unsigned long long>("hot_best", 2);
        unsigned long long init[2] = {0, ~0ull};
        STG_CUDA(cudaMemcpyAsync(best, init, 16, cudaMemcpyHostToDevice, st));
        for (int pass = 0; pass < 2; ++pass)
            LAUNCH(k_hottest, grid_for(m.n * 32), kThreads, m.n, nullptr, m.cnt, 1, m.dn_off, m.dn, key, pass, best);
        unsigned long long hb[2];
        down(hb, best, 2);
        if (hb[1] == ~0ull) return {};
        uint32_t g;
        down(&g, merged_rep + hb[1], 1);
        uint64_t o[2];
        down(o, m.off + g, 2);
        std::vector<uint32_t> ks(o[1] - o[0]);
        down(ks.data(), m.arena + o[0], ks.size());
        std::vector<std::string> out;
        for (uint32_t k : ks) out.push_back(gname(k));
        return out;
    }
    std::vector<int32_t> all_cpu_ranks() {
        std::vector<uint8_t> mine;
        for (int32_t r : res.cpu_rank_ids) put<int32_t>(mine, r);
        std::vector<int32_t> out;
        for (const auto& b : allgather_bytes(mine))
            for (const uint8_t* p = b.data(); p < b.data() + b.size();) out.push_back(get<int32_t>(p));
        std::sort(out.begin(), out.end());
        return out;
    }

    void diagnose() {
        Report& rep = res.report;
        rep = Report{};
        // detect_straggler alerts (diagnosis.cpp:97-110)
        std::vector<int> alerts;
        for (int32_t r = 0; r < span; ++r)
            if (res.flag_count[r] && res.flag_count[r] * 2 > res.n_windowed) alerts.push_back(r);
        if (!alerts.empty()) {
            rep.flagged_ranks = alerts;  // already ascending
            // median_lateness_rank (diagnosis.cpp:284-297)
            std::vector<std::pair<double, int>> means;
            for (int32_t r = 0; r < span; ++r)
                if (res.lat_present[r] && !std::binary_search(alerts.begin(), alerts.end(), r))
                    means.emplace_back(res.mean_lat_all[r], r);
            if (means.empty()) {
                rep.verdict = STG_VERDICT_INCONCLUSIVE;
                rep.notes.push_back("no reference rank available");
                return;
            }
            std::sort(means.begin(), means.end());
            int ref = means[means.size() / 2].second;
            rep.reference_rank = ref;
            int strag = alerts.front();
            int concluded = STG_VERDICT_INCONCLUSIVE;
            std::vector<Evidence> gpu_ev, cpu_ev, os_ev;
            // GPU layer (gpu_diff diagnosis.cpp:122-172)
            if (res.gpu.count(strag) && res.gpu.count(ref)) {
                const auto& S_ = res.gpu.at(strag);
                const auto& Rf = res.gpu.at(ref);
                std::vector<double> slow;
                std::map<std::string, double> slowdown;
                int64_t total_added = 0;
                std::string top;
                std::string prefix = cfg.gpu_exclude_prefix;
                for (const auto& [name, t_ref] : Rf) {
                    if (t_ref < cfg.gpu_ref_floor_ns) continue;
                    if (!prefix.empty() && name.rfind(prefix, 0) == 0) continue;
                    auto it = S_.find(name);
                    if (it == S_.end()) continue;
                    double s = double(it->second) / double(t_ref) - 1.0;
                    slowdown[name] = s;
                    slow.push_back(s);
                    int64_t added = it->second - t_ref;
                    if (added > 0) {
                        total_added += added;
                        if (top.empty() || added > S_.at(top) - Rf.at(top)) top = name;
                    }
                }
                int gv = 0;  // None
                if (!slow.empty()) {
                    double med = median_of(slow);
                    double mu = mean_of(slow);
                    double sg = pstd(slow, mu);
                    double cv = mu != 0.0 ? std::fabs(sg / mu) : 0.0;
                    double share = 0.0;
                    if (!top.empty() && total_added > 0) share = double(S_.at(top) - Rf.at(top)) / double(total_added);
                    if (med <= cfg.gpu_median_none) gv = 0;
                    else if (med > cfg.gpu_median_uniform && cv < cfg.gpu_cv_uniform) gv = 1;
                    else if (share > cfg.gpu_top_share_specific) gv = 2;
                }
                for (const auto& [name, s] : slowdown)
                    gpu_ev.push_back({"gpu", name, double(S_.at(name)), double(Rf.at(name)), s});
                if (gv == 1) concluded = STG_VERDICT_GPU_UNIFORM;
                else if (gv == 2) {
                    concluded = STG_VERDICT_GPU_SPECIFIC;
                    rep.top_path = {top};
                }
            } else {
                rep.notes.push_back("gpu profiles missing; gpu layer skipped");
            }
            // CPU layer (cpu_diff diagnosis.cpp:177-208)
            int is = cpu_index(strag), iq = cpu_index(ref);
            if (dist()) {
                mark("d:enter");
                global_names();
                mark("d:names");
                cpu_owners();
                mark("d:owners");
                const int os_ = cpu_owner[size_t(strag)], oq = cpu_owner[size_t(ref)];
                if (os_ >= 0 && oq >= 0) {
                    // candidates first (as on one GPU): d = fs - fr <= fs, so the
                    // straggler's owner sums exact fractions only for names whose
                    // own estimate can exceed delta; the reference's owner then adds
                    // the exact fractions of those names; both lists are small
                    inclusive_counts();
                    if (F) dense_name(0);  // h_dense_final
                    std::vector<uint32_t> dense_of;
                    std::vector<std::pair<uint32_t, double>> fs_, fr_;
                    std::vector<uint8_t> bS, bR;
                    if (c.wrank == os_) {
                        const int si = cpu_index(strag);
                        uint64_t lo[2];
                        down(lo, d_line_off + si, 2);
                        const double margin = double(lo[1] - lo[0] + 8) * std::ldexp(1.0, -50);
                        uint8_t* want = dev<uint8_t>("xf_want", std::max<uint64_t>(F, 1));
                        if (F)
                            LAUNCH(k_frac_want, grid_for(F), kThreads, F, d_incl + uint64_t(si) * F,
                                   double(h_n_in[size_t(si)]), cfg.delta - margin, want);
                        auto fr2 = exact_fractions2(lo[0], lo[1] - lo[0], h_n_in[size_t(si)], 0, 0, 0, false, nullptr,
                                                    nullptr, nullptr, want);
                        for (const auto& [f, v] : fr2[0]) {
                            put<uint32_t>(bS, to_global(h_dense_final[f]));
                            put<double>(bS, v);
                            dense_of.push_back(f);
                        }
                    }
                    bS = bcast_bytes(std::move(bS), os_);
                    for (const uint8_t* p = bS.data(); p < bS.data() + bS.size();) {
                        const uint32_t k = get<uint32_t>(p);
                        fs_.emplace_back(k, get<double>(p));
                    }
                    mark("d:fracs");
                    if (c.wrank == oq) {
                        const int ri = cpu_index(ref);
                        std::vector<uint8_t> want(std::max<uint64_t>(F, 1), 0);
                        bool any = false;
                        for (const auto& [g, v] : fs_) {
                            const int64_t f = dense_of_global(g);
                            if (f >= 0) {
                                want[size_t(f)] = 1;
                                any = true;
                            }
                        }
                        if (any) {
                            uint64_t lo[2];
                            down(lo, d_line_off + ri, 2);
                            const uint8_t* d_want = up<uint8_t>("xf_want", want.data(), want.size());
                            auto fr2 = exact_fractions2(lo[0], lo[1] - lo[0], h_n_in[size_t(ri)], 0, 0, 0, false,
                                                        nullptr, nullptr, nullptr, d_want);
                            for (const auto& [f, v] : fr2[0]) {
                                put<uint32_t>(bR, to_global(h_dense_final[f]));
                                put<double>(bR, v);
                            }
                        }
                    }
                    bR = bcast_bytes(std::move(bR), oq);
                    for (const uint8_t* p = bR.data(); p < bR.data() + bR.size();) {
                        const uint32_t k = get<uint32_t>(p);
                        fr_.emplace_back(k, get<double>(p));
                    }
                    mark("d:bcast");
                    struct Cand { std::string fn; double fs, fr, d; uint32_t key; };
                    std::vector<Cand> cands;
                    size_t j = 0;
                    for (const auto& [k, fs] : fs_) {  // key order == name order
                        while (j < fr_.size() && fr_[j].first < k) ++j;
                        double fr = j < fr_.size() && fr_[j].first == k ? fr_[j].second : 0.0;
                        double d = fs - fr;
                        if (d > cfg.delta) cands.push_back({gname(k), fs, fr, d, k});
                    }
                    std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
                        return a.d != b.d ? a.d > b.d : a.fn < b.fn;
                    });
                    for (const auto& cd : cands) cpu_ev.push_back({"cpu", cd.fn, cd.fs, cd.fr, cd.d});
                    if (concluded == STG_VERDICT_INCONCLUSIVE && !cands.empty()) {
                        concluded = STG_VERDICT_CPU_INTERFERENCE;
                        std::vector<std::string> path;
                        if (c.wrank == os_) {
                            uint64_t lo[2];
                            down(lo, d_line_off + is, 2);
                            auto it = std::lower_bound(fs_.begin(), fs_.end(), std::make_pair(cands.front().key, -1e300));
                            path = hottest(lo[0], lo[1], dense_of[size_t(it - fs_.begin())], false);
                        }
                        rep.top_path = bcast_path(std::move(path), os_);
                        mark("d:path");
                    }
                } else {
                    rep.notes.push_back("cpu profiles missing; cpu layer skipped");
                }
            } else if (is >= 0 && iq >= 0) {
                struct Cand { std::string fn; double fs, fr, d; uint32_t f; };
                std::vector<Cand> cands;
                std::vector<uint64_t> loff(size_t(R) + 1);
                down(loff.data(), d_line_off, loff.size());
                const uint64_t lo[2] = {loff[size_t(is)], loff[size_t(is) + 1]};
                const uint64_t lo2[2] = {loff[size_t(iq)], loff[size_t(iq) + 1]};
                // Candidates first: fs and fr are sequential double sums of
                // count/total over <= n lines each (folded.cpp:45-54), so each is
                // within (n + 2) * 2^-52 of its exact-integer estimate inc/total.
                // Names whose estimated d stays below delta by more than the sum
                // of both bounds cannot pass d > delta; the rest get the exact
                // line-order sums (the values the report carries).
                inclusive_counts();
                uint8_t* want = dev<uint8_t>("xf_want", std::max<uint64_t>(F, 1));
                const double margin = double((lo[1] - lo[0]) + (lo2[1] - lo2[0]) + 8) * std::ldexp(1.0, -50);
                LAUNCH(k_diff_cands, grid_for(F), kThreads, F, d_incl, uint32_t(R), uint32_t(is), uint32_t(iq),
                       double(h_n_in[is]), double(h_n_in[iq]), cfg.delta - margin, want);
                auto both = exact_fractions2(lo[0], lo[1] - lo[0], h_n_in[is], lo2[0], lo2[1] - lo2[0], h_n_in[iq],
                                             false, nullptr, nullptr, nullptr, want);
                mark("d:fracs2");
                const auto& fs_ = both[0];
                const auto& fr_ = both[1];
                size_t j = 0;
                for (const auto& [f, fs] : fs_) {  // name order (dense index order)
                    while (j < fr_.size() && fr_[j].first < f) ++j;
                    double fr = j < fr_.size() && fr_[j].first == f ? fr_[j].second : 0.0;
                    double d = fs - fr;
                    if (d > cfg.delta) cands.push_back({std::string(), fs, fr, d, f});
                }
                {
                    std::vector<uint32_t> want;
                    want.reserve(cands.size());
                    for (const auto& cd : cands) want.push_back(cd.f);
                    auto nm = dense_names(want);
                    for (size_t k = 0; k < cands.size(); ++k) cands[k].fn = std::move(nm[k]);
                }
                std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
                    return a.d != b.d ? a.d > b.d : a.fn < b.fn;
                });
                for (const auto& cd : cands) cpu_ev.push_back({"cpu", cd.fn, cd.fs, cd.fr, cd.d});
                if (concluded == STG_VERDICT_INCONCLUSIVE && !cands.empty()) {
                    concluded = STG_VERDICT_CPU_INTERFERENCE;
                    rep.top_path = hottest(lo[0], lo[1], cands.front().f, false);
                    mark("d:hottest");
                }
            } else {
                rep.notes.push_back("cpu profiles missing; cpu layer skipped");
            }
            // OS layer (os_diff diagnosis.cpp:213-243)
            if (res.os.count(strag) && res.os.count(ref)) {
                const OsAcc& s = res.os.at(strag);
                const OsAcc& r = res.os.at(ref);
                auto check = [&](const std::string& name, int64_t sv, int64_t rv, int64_t floor) {
                    if (sv - rv < floor) return;
                    if (rv == 0) {
                        os_ev.push_back({"os", name, double(sv), double(rv), 0.0});
                        return;
                    }
                    double ratio = double(sv) / double(rv);
                    if (ratio >= cfg.os_min_ratio) os_ev.push_back({"os", name, double(sv), double(rv), ratio});
                };
                for (const auto& [k, v] : s.interrupts) {
                    auto it = r.interrupts.find(k);
                    check("interrupt:" + k, v, it == r.interrupts.end() ? 0 : it->second, cfg.os_interrupt_floor);
                }
                for (const auto& [k, v] : s.softirqs) {
                    auto it = r.softirqs.find(k);
                    check("softirq:" + k, v, it == r.softirqs.end() ? 0 : it->second, cfg.os_interrupt_floor);
                }
                check("sched_delay_p99_ns", s.p99, r.p99, cfg.os_sched_delay_floor_ns);
                check("numa_migrations", s.migrations, r.migrations, cfg.os_migration_floor);
                if (concluded == STG_VERDICT_INCONCLUSIVE && !os_ev.empty()) concluded = STG_VERDICT_OS_INTERFERENCE;
            } else {
                rep.notes.push_back("os snapshots missing; os layer skipped");
            }
            rep.verdict = concluded;
            for (auto* v : {&gpu_ev, &cpu_ev, &os_ev}) rep.evidence.insert(rep.evidence.end(), v->begin(), v->end());
            if (rep.verdict == STG_VERDICT_INCONCLUSIVE) rep.notes.push_back("straggler detected but no layer concluded");
            return;
        }
        // No straggler: temporal route (diagnosis.cpp:383-428)
        if (res.has_baseline_iteration && !res.iteration_times_ms.empty()) {
            double now = mean_of(res.iteration_times_ms);
            double base = res.baseline_iteration_ms;
            if (base > 0.0 && now > base * (1.0 + cfg.iteration_regression_gate)) {
                if (!res.has_baseline) {
                    rep.verdict = STG_VERDICT_INCONCLUSIVE;
                    rep.notes.push_back("iteration time regressed but no baseline profile");
                    return;
                }
                struct Cand { std::string fn; double now, base, d; uint32_t f; };
                std::vector<Cand> cands;
                if (dist()) {
                    global_names();
                    MergedSeqs m = merged_union();
                    if (m.n)
                        for (const auto& [k, nw] : exact_fractions(0, m.n, m.total, true, m.dn_off, m.dn, m.cnt)) {
                            std::string fn = gname(k);
                            auto it = res.baseline.find(fn);
                            double b = it == res.baseline.end() ? 0.0 : it->second;
                            double d = nw - b;
                            if (d > res.baseline_delta) cands.push_back({fn, nw, b, d, k});
                        }
                    std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
                        return a.d != b.d ? a.d > b.d : a.fn < b.fn;
                    });
                    auto ranks = all_cpu_ranks();
                    if (!cands.empty()) {
                        rep.verdict = STG_VERDICT_TEMPORAL;
                        rep.flagged_ranks.assign(ranks.begin(), ranks.end());
                        for (const auto& cd : cands) rep.evidence.push_back({"temporal", cd.fn, cd.now, cd.base, cd.d});
                        rep.top_path = merged_path(m, cands.front().f);
                        return;
                    }
                    rep.verdict = STG_VERDICT_INCONCLUSIVE;
                    rep.notes.push_back("iteration time regressed but no profile delta above delta");
                    return;
                }
                if (F > 0) {
                    auto sc = dev<unsigned long long>("seq_counts", S);
                    zero(sc, S * 8);
                    LAUNCH(k_seq_counts, grid_for(L), kThreads, L, d_lkey, d_lcount, sc);
                    uint64_t T = 0;
                    for (uint64_t t : res.cpu_totals) T += t;
                    for (const auto& [f, nw] : exact_fractions(0, S, T, true)) {
                        std::string fn = dense_name(f);
                        auto it = res.baseline.find(fn);
                        double b = it == res.baseline.end() ? 0.0 : it->second;
                        double d = nw - b;
                        if (d > res.baseline_delta) cands.push_back({fn, nw, b, d, f});
                    }
                }
                std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
                    return a.d != b.d ? a.d > b.d : a.fn < b.fn;
                });
                if (!cands.empty()) {
                    rep.verdict = STG_VERDICT_TEMPORAL;
                    rep.flagged_ranks.assign(res.cpu_rank_ids.begin(), res.cpu_rank_ids.end());
                    for (const auto& cd : cands) rep.evidence.push_back({"temporal", cd.fn, cd.now, cd.base, cd.d});
                    rep.top_path = hottest(0, 0, cands.front().f, true);
                    return;
                }
                rep.verdict = STG_VERDICT_INCONCLUSIVE;
                rep.notes.push_back("iteration time regressed but no profile delta above delta");
                return;
            }
        }
        rep.verdict = STG_VERDICT_HEALTHY;
    }

    // ------------------------------------------------------ waterline
    // compute_waterline + flag_ranks over the window's CPU profiles.
    void waterline_dist() {
        res.waterline_done = true;
        inclusive_counts();
        global_names();
        const size_t nr = res.cpu_rank_ids.size();
        unsigned long long* drt = dev<unsigned long long>("wl_rt", 1);
        unsigned long long nrl = nr;
        STG_CUDA(cudaMemcpyAsync(drt, &nrl, 8, cudaMemcpyHostToDevice, st));
        nccl(ncclAllReduce(drt, drt, 1, ncclUint64, ncclSum, comm(), st));
        const uint64_t RT = get1(drt);
        mark("w:ranks");
        if (RT < 2) {
            res.waterline_json = "{\"error\": \"waterline requires at least 2 ranks\"}";
            return;
        }
        // per-name sums only over the names some GPU's profiles use: the sorted
        // union of the contexts' global keys (not the whole dictionary)
        // dense name -> global key on the device (to_global, one thread per name)
        uint32_t* d_gkey = dev<uint32_t>("wl_gkey_g", std::max<uint64_t>(F, 1));
        if (F) {
            const uint64_t nl = gn.loc_final.size(), ng = gn.pos.size();
            // (empty label lists: nothing is copied, the kernel does not read them)
            const uint64_t* d_lf = up<uint64_t>("tg_lf", gn.loc_final.data(), nl);
            const uint32_t* d_lg = up<uint32_t>("tg_lg", gn.loc_global.data(), nl);
            const uint32_t* d_ps = up<uint32_t>("tg_ps", gn.pos.data(), ng);
            LAUNCH(k_to_global, grid_for(F), kThreads, F, d_dense_final, d_lf, d_lg, nl, d_ps, ng, d_gkey);
        }
        // used-name byte map over the global name space, OR-ed over the group
        // (all-reduce max), scanned into compact indices on the device
        const uint64_t NGF = c.dict.size() + gn.lab.size();
        uint8_t* umap = dev<uint8_t>("wl_umap", NGF);
        zero(umap, NGF);
        if (F) LAUNCH(k_mark_u8, grid_for(F), kThreads, F, d_gkey, umap);
        nccl(ncclAllReduce(umap, umap, NGF, ncclUint8, ncclMax, comm(), st));
        uint32_t* u32 = dev<uint32_t>("wl_u32", NGF + 1);
        uint32_t* uscan = dev<uint32_t>("wl_uscan", NGF + 1);
        LAUNCH(k_u8_to_u32, grid_for(NGF + 1), kThreads, NGF, umap, u32);
        excl_sum(u32, uscan, NGF + 1);
        const uint64_t NU = get1(uscan + NGF);
        mark("w:union");
        uint32_t* d_gk = dev<uint32_t>("wl_gkey", std::max<uint64_t>(F, 1));
        if (F) LAUNCH(k_gather_u32, grid_for(F), kThreads, F, d_gkey, uscan, d_gk);
        const uint64_t NG = std::max<uint64_t>(NU, 1);
        double* s1 = dev<double>("wl_s1", NG);
        unsigned* np = dev<unsigned>("wl_np", NG);
        double* s2 = dev<double>("wl_s2", NG);
        zero(s1, NG * 8);
        zero(np, NG * 4);
        zero(s2, NG * 8);

        uint32_t* rows = up<uint32_t>("wl_rows", res.cpu_rank_index.data(), nr);
        if (F && nr) LAUNCH(k_wl_pass1, grid_for(F * 32), kThreads, F, rows, int(nr), d_incl, d_totals, d_gk, s1, np);
        nccl(ncclAllReduce(s1, s1, NG, ncclFloat64, ncclSum, comm(), st));
        nccl(ncclAllReduce(np, np, NG, ncclUint32, ncclSum, comm(), st));
        if (F && nr) LAUNCH(k_wl_pass2, grid_for(F * 32), kThreads, F, rows, int(nr), d_incl, d_totals, d_gk, s1, np, double(RT), s2);
        nccl(ncclAllReduce(s2, s2, NG, ncclFloat64, ncclSum, comm(), st));
        mark("w:sums");
        double* mean = dev<double>("wlg_mean", NG);
        double* sd = dev<double>("wlg_sd", NG);
        LAUNCH(k_wl_final, grid_for(NG), kThreads, NG, s1, np, s2, double(RT), mean, sd);
        unsigned long long cap = std::max<uint64_t>(1, std::min<uint64_t>(F * std::max<size_t>(nr, 1), 1u << 24));
        uint32_t* o_r = dev<uint32_t>("wl_or", cap);
        uint32_t* o_f = dev<uint32_t>("wl_of", cap);
        double* o_fr = dev<double>("wl_ofr", cap);
        double* o_th = dev<double>("wl_oth", cap);
        unsigned long long* n_out = dev<unsigned long long>("wl_n", 1);
        zero(n_out, 8);
        if (F && nr)
            LAUNCH(k_flag_g, grid_for(F * nr), kThreads, F, rows, int(nr), d_incl, d_totals, cfg.k, d_gk, mean, sd, o_r,
                   o_f, o_fr, o_th, n_out, cap);
        res.wl_flags = std::min<uint64_t>(get1(n_out), cap);
        res.wl_F = F;
        res.wl_dist = true;
        res.wl_NG = NU;
        res.wl_NGF = NGF;
        res.g_lab_final = gn.lab_final;
        res.g_lab = gn.lab;
        res.waterline_json.clear();  // rendered on request
    }

    void waterline() {
        res.wl_dist = false;
        if (dist()) return waterline_dist();
        res.waterline_done = true;
        std::string out;
        size_t nr = res.cpu_rank_ids.size();
        if (nr < 2) {
            res.waterline_json = "{\"error\": \"waterline requires at least 2 ranks\"}";
            return;
        }
        inclusive_counts();
        uint32_t* rows = up<uint32_t>("wl_rows", res.cpu_rank_index.data(), nr);
        double* mean = dev<double>("wl_mean", F);
        double* sd = dev<double>("wl_sd", F);
        uint8_t* pres = dev<uint8_t>("wl_pres", F);
        LAUNCH(k_waterline, grid_for(F * 32), kThreads, F, rows, int(nr), d_incl, d_totals, mean, sd, pres);
        unsigned long long cap = std::max<uint64_t>(1, std::min<uint64_t>(F * nr, 1u << 24));
        uint32_t* o_r = dev<uint32_t>("wl_or", cap);
        uint32_t* o_f = dev<uint32_t>("wl_of", cap);
        double* o_fr = dev<double>("wl_ofr", cap);
        double* o_th = dev<double>("wl_oth", cap);
        unsigned long long* n_out = dev<unsigned long long>("wl_n", 1);
        zero(n_out, 8);
        LAUNCH(k_flag, grid_for(F * nr), kThreads, F, rows, int(nr), d_incl, d_totals, cfg.k, mean, sd, o_r, o_f, o_fr,
               o_th, n_out, cap);
        res.wl_flags = std::min<uint64_t>(get1(n_out), cap);
        res.wl_F = F;
        res.waterline_json.clear();  // rendered on request (waterline_json())
    }

    // Distributed error agreement.  Input errors found on one context's shard
    // (an empty stack, a timestamp regression, ...) must not leave the other
    // contexts waiting in the next collective: every context runs the local
    // stage, then all agree on the first failure in reference order — stage
    // (collectives, then the CPU rank loop, then the GPU/OS loops of
    // build_group_data, bundle.cpp:252-324), then the lowest failing rank —
    // and all throw the owner's exact error.
    int err_stage = 0;
    template <class F>
    void agreed(F&& f) {
        if (!dist()) {
            f();
            return;
        }
        long long key = LLONG_MAX;
        int code = STG_OK;
        std::string msg;
        try {
            f();
        } catch (const Error& e) {
            code = e.code;
            msg = e.what();
        } catch (const std::exception& e) {
            code = STG_ENOMEM;
            msg = e.what();
        }
        if (code != STG_OK)
            key = ((long long)err_stage << 48) | ((long long)(fail_rank + 1) << 8) | (long long)c.wrank;
        long long* d = dev<long long>("dx_err", 1);
        STG_CUDA(cudaMemcpyAsync(d, &key, 8, cudaMemcpyHostToDevice, st));
        nccl(ncclAllReduce(d, d, 1, ncclInt64, ncclMin, comm(), st));
        key = get1(d);
        if (key == LLONG_MAX) return;
        const int owner = int(key & 0xff);
        std::vector<uint8_t> b;
        if (c.wrank == owner) {
            put<int32_t>(b, code);
            put_str(b, msg);
        }
        b = bcast_bytes(std::move(b), owner);
        const uint8_t* q = b.data();
        const int32_t oc = get<int32_t>(q);
        fail(oc, get_str(q));
    }

    // STG_TRACE=1: host wall time per stage on stderr
    bool trace = std::getenv("STG_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t_last = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!trace) return;
        auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[stg] r%d %-12s %8.3f ms  syncs %3u launches %3u  @%.3f\n", c.wrank, what,
                     std::chrono::duration<double, std::milli>(now - t_last).count(), syncs, launches,
                     std::fmod(std::chrono::duration<double, std::milli>(now.time_since_epoch()).count(), 1e5));
        t_last = now;
    }

    void run() {
        mark("start");
        res.group = w.group;
        // a LoadedBundle always carries a baseline (bundle.hpp:37-38), which
        // build_group_data copies (bundle.cpp:257-258): empty / 0.0 if absent
        res.has_baseline = true;
        res.baseline_delta = w.has_baseline ? w.baseline_delta : 0.005;
        res.baseline.clear();
        for (uint32_t i = 0; i < w.n_baseline; ++i) res.baseline[w.baseline_names[i]] = w.baseline_fracs[i];
        res.has_baseline_iteration = true;
        res.baseline_iteration_ms = w.has_baseline_iteration ? w.baseline_iteration_ms : 0.0;
        cudaEventRecord(ev[0], st);
        agreed([&] { rank_space(); });
        rank_span_agree();
        mark("rank_space");
        agreed([&] { coll_result_init(); });
        n_coll_all = w.n_coll;
        if (coll_sharded()) {  // local half may fail (agreed), the exchange does not
            agreed([&] {
                err_stage = 0;
                coll_local();
            });
            coll_exchange();
        }
        agreed([&] {
            err_stage = 0;
            if (!coll_sharded()) collectives();
            cudaEventRecord(ev[1], st);
            mark("collectives");
            err_stage = 1;
            samples();  // runs gpu_os() on the side stream while k_sym_agg streams
            err_stage = 2;
            if (!gpu_os_done) gpu_os();
        });
        if (side_coll_tail(false)) cudaEventRecord(ev[1], st);  // no samples stage: stage d ends here
        if (side_sharded()) gpu_os_reduce();
        mark("samples+fold");
        if (ev_unset_fold()) {
            cudaEventRecord(ev[2], st);
            cudaEventRecord(ev[3], st);
            cudaEventRecord(ev[4], st);
            cudaEventRecord(ev[5], st);
            cudaEventRecord(ev[6], st);
        }
        diagnose();
        mark("diagnose");
        res.waterline_done = false;
        if (cfg.want_waterline) waterline();
        mark("waterline");
        cudaEventRecord(ev[7], st);
        STG_CUDA(cudaStreamSynchronize(st));
        stg_run_stats& s = res.stats;
        s = stg_run_stats{};
        uint64_t nin = 0;
        for (uint64_t t : res.cpu_totals) nin += t;
        s.n_samples_in_window = nin;
        s.n_lines = res.n_lines;
        s.n_sequences = res.n_seq;
        s.n_names = res.n_names;
        s.n_unknown = res.n_unknown;
        s.n_instances = res.n_instances;
        s.n_windowed = res.n_windowed;
        s.n_cpu_ranks = res.cpu_rank_ids.size();
        s.verdict = res.report.verdict;
        s.n_flagged = int32_t(res.report.flagged_ranks.size());
        cudaEventElapsedTime(&s.ms_collectives, ev[0], ev[1]);
        cudaEventElapsedTime(&s.ms_symbolize, ev[2], ev[3]);
        cudaEventElapsedTime(&s.ms_fold, ev[4], ev[5]);
        cudaEventElapsedTime(&s.ms_diff, ev[5], ev[6]);
        cudaEventElapsedTime(&s.ms_total, ev[0], ev[7]);
        s.h2d_bytes = h2d;
        s.d2h_bytes = d2h;
        s.kernel_launches = launches;
        s.agg_attempts = uint32_t(res.agg_attempts);
        s.prefix_hits = res.pfx_hits;
        s.prefix_misses = res.pfx_misses;
        s.verified = res.verified;
        s.verify_retries = res.verify_retries;
        mark("stats");
    }
    bool ev_unset_fold() const { return R == 0 || L == 0; }
};

}  // namespace stg
