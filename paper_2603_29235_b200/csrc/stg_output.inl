// stg_output.inl — resolve verb and result renderings (included by stg_window.cu).
namespace stg {

static const char* kVerdictNames[] = {"healthy",        "gpu-uniform-slowdown", "gpu-specific-kernel",
                                      "cpu-interference", "os-interference",   "temporal-degradation",
                                      "inconclusive"};

// resolve_stacks (symrepo.cpp:122-143) as one batched GPU lookup.
void run_resolve(Ctx& c, Result& res, uint64_t n, const uint64_t* pc, const uint16_t* bin, int32_t n_bins,
                 const uint8_t* ids, int mode, uint32_t* out) {
    stg_window w{};
    w.n_bins = n_bins;
    w.bin_build_ids = ids;
    stg_config cfg{};
    stg_config_default(&cfg);
    cfg.lookup_mode = mode;
    Runner rn(c, w, cfg, res);
    symtab_refresh_dictionary(c);
    std::vector<DevTable> tabs(std::max<int32_t>(n_bins, 1));
    for (int32_t b = 0; b < n_bins; ++b) {
        DevTable& t = tabs[size_t(b)];
        std::memset(&t, 0, sizeof t);
        auto it = c.table_by_id.find(std::string(reinterpret_cast<const char*>(ids + 20 * b), 20));
        if (it == c.table_by_id.end()) continue;
        HostTable& h = *c.tables[it->second];
        if (h.n == 0) continue;
        t = DevTable{h.d_e, h.d_bucket, h.first_start, h.last_start, h.shift, h.nb, h.n, 1};
    }
    DevTable* d_tabs = rn.up<DevTable>("rv_tabs", tabs.data(), tabs.size());
    const uint64_t* d_pc = rn.up<uint64_t>("rv_pc", pc, n);
    const uint16_t* d_bin = rn.up<uint16_t>("rv_bin", bin, n);
    uint32_t* d_out = rn.dev<uint32_t>("rv_out", n);
    uint32_t cap = uint32_t(std::max<uint64_t>(1024, next_pow2(2 * n + 2)));
    UnkSlot* unk = rn.dev<UnkSlot>("rv_unk", cap);
    rn.zero(unk, size_t(cap) * sizeof(UnkSlot));
    unsigned* used = rn.dev<unsigned>("rv_used", 1);
    int* ovf = rn.dev<int>("rv_ovf", 1);
    int* ebin = rn.dev<int>("rv_ebin", 1);
    rn.zero(used, 4);
    rn.zero(ovf, 4);
    rn.zero(ebin, 4);
    cudaStream_t st = c.stream;
    uint32_t& launches = rn.launches;
    if (n) LAUNCH(k_resolve, grid_for(n), kThreads, n, d_pc, d_bin, d_tabs, uint32_t(n_bins), mode,
                  UnkSet{unk, cap - 1, cap, used, ovf}, ebin, d_out);
    if (rn.get1(ebin)) fail(STG_EINVAL, "frame binary index out of range");
    if (rn.get1(ovf)) fail(STG_ENOMEM, "unknown-frame set overflow");
    ulonglong2* u_rec = rn.dev<ulonglong2>("rv_urec", cap);
    unsigned* nu = rn.dev<unsigned>("rv_nu", 1);
    rn.zero(nu, 4);
    LAUNCH(k_unk_compact, grid_for(cap), kThreads, cap, unk, u_rec, nu);
    uint32_t NU = rn.get1(nu);
    std::vector<ulonglong2> ur(NU);
    rn.down(ur.data(), u_rec, NU);
    std::vector<uint32_t> hs(NU), hb(NU);
    std::vector<uint64_t> hp(NU);
    for (uint32_t k = 0; k < NU; ++k) {
        hp[k] = ur[k].x;
        hs[k] = uint32_t(ur[k].y);
        hb[k] = uint32_t(ur[k].y >> 32);
    }
    rn.merge_labels(NU, hs, hb, hp, cap);
    if (n) {
        LAUNCH(k_remap, grid_for(n), kThreads, n, d_out, static_cast<const uint32_t*>(c.buf("u_final").p),
               static_cast<const uint32_t*>(c.buf("u_pos").p), uint32_t(rn.n_pos));
        rn.down(out, d_out, n);
    }
    res.n_names = c.dict.size() + res.unk_labels.size();
}

// DiagnosisReport::to_json (diagnosis.cpp:437-455): nlohmann dump(2), the same bytes
std::string report_json(Ctx& c) { return report_json_dump2(c.result->report); }
std::string report_text_of(Ctx& c) { return report_text(c.result->report); }

template <class T>
static void d2h(Ctx& c, T* host, const char* name, size_t n, size_t offset = 0) {
    if (!n) return;
    const T* d = static_cast<const T*>(c.buf(name).p) + offset;
    STG_CUDA(cudaMemcpyAsync(host, d, n * sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    STG_CUDA(cudaStreamSynchronize(c.stream));
}

// Lines of CPU rank i: (sequence name keys, count), in folded order.
// The folded lines of the last window on the host, one bulk download per result.
static const Result::HostFold& host_fold(Ctx& c) {
    Result& r = *c.result;
    Result::HostFold& h = r.hf;
    if (h.ok) return h;
    h.lkey.resize(r.n_lines);
    h.lcount.resize(r.n_lines);
    h.dense_rep.resize(r.n_seq);
    h.line_off.assign(size_t(r.n_window_ranks) + 1, 0);
    if (r.n_lines) {
        d2h(c, h.lkey.data(), "lkey_s", r.n_lines);
        d2h(c, h.lcount.data(), "lcount_s", r.n_lines);
        d2h(c, h.dense_rep.data(), "dense_rep", r.n_seq);
        h.seq_off.resize(r.n_gid + 1);
        d2h(c, h.seq_off.data(), "seq_off", r.n_gid + 1);
        h.arena.resize(h.seq_off[r.n_gid]);
        d2h(c, h.arena.data(), "arena", h.arena.size());
        d2h(c, h.line_off.data(), "line_off", h.line_off.size());
    }
    h.ok = true;
    return h;
}

// Lines of CPU rank i: (sequence name keys, count), in folded order.
void rank_lines(Ctx& c, uint32_t i, std::vector<uint64_t>& key_off, std::vector<uint32_t>& keys,
                std::vector<uint64_t>& counts) {
    Result& r = *c.result;
    const uint32_t row = r.cpu_rank_index.at(i);
    const Result::HostFold& h = host_fold(c);
    key_off.assign(1, 0);
    keys.clear();
    counts.clear();
    if (!r.n_lines) return;
    for (uint64_t l = h.line_off[row]; l < h.line_off[row + 1]; ++l) {
        const uint32_t g = h.dense_rep[uint32_t(h.lkey[l])];
        keys.insert(keys.end(), h.arena.begin() + h.seq_off[g], h.arena.begin() + h.seq_off[g + 1]);
        key_off.push_back(keys.size());
        counts.push_back(h.lcount[l]);
    }
}

// ---- flame graphs (render_flamegraph / render_diff_flamegraph, svg.cpp:157-172)
// The reference builds a std::map trie of the profile's lines and renders it
// depth first.  The lines are already in std::map order here, so the trie's
// pre-order is one pass over them (a new node wherever a line leaves the
// previous line's prefix, counts summed over the contiguous run of lines that
// share it), and the layout is the reference's own sequence of double
// operations (widths and sibling offsets accumulated left to right), printed
// with the same ostream formatting.
namespace svg {
struct Node {
    uint32_t depth;
    uint32_t key;
    uint64_t before, after;
};
static std::string escape(const std::string& s) {
    std::string out;
    for (char ch : s) {
        switch (ch) {
            case '&': out += "&amp;"; break;
            case '<': out += "&lt;"; break;
            case '>': out += "&gt;"; break;
            case '"': out += "&quot;"; break;
            default: out += ch;
        }
    }
    return out;
}
static std::string name_color(const std::string& name) {
    uint64_t h = 1469598103934665603ull;
    for (char ch : name) {
        h ^= uint8_t(ch);
        h *= 1099511628211ull;
    }
    std::ostringstream os;
    os << "rgb(" << 205 + int(h % 50) << "," << int(h / 50 % 180) << "," << int(h / 9000 % 55) << ")";
    return os.str();
}
static std::string diff_color(uint64_t before, uint64_t after, uint64_t tb, uint64_t ta) {
    const double fb = tb ? double(before) / double(tb) : 0.0;
    const double fa = ta ? double(after) / double(ta) : 0.0;
    const double delta = fa - fb;
    std::ostringstream os;
    if (delta > 0.0005) {
        const int shade = 255 - std::min(155, int(delta * 4000));
        os << "rgb(255," << shade << "," << shade << ")";
    } else if (delta < -0.0005) {
        const int shade = 255 - std::min(155, int(-delta * 4000));
        os << "rgb(" << shade << "," << shade << ",255)";
    } else {
        os << "rgb(224,224,224)";
    }
    return os.str();
}
}  // namespace svg

// kind 0: one rank's profile; kind 1: diff (before = rank_a, after = rank_b)
std::string flamegraph_svg(Ctx& c, int kind, int32_t rank_a, int32_t rank_b, const stg_svg_options& o) {
    Result& r = *c.result;
    auto index_of = [&](int32_t rank) {
        auto it = std::lower_bound(r.cpu_rank_ids.begin(), r.cpu_rank_ids.end(), rank);
        if (it == r.cpu_rank_ids.end() || *it != rank) fail(STG_EINVAL, "unknown rank id: " + std::to_string(rank));
        return uint32_t(it - r.cpu_rank_ids.begin());
    };
    const Result::HostFold& h = host_fold(c);
    // the (before, after) line list in map order: one rank, or the merge of two
    // (lines of both ranks carry global sequence ranks, so merging by them is
    // merging by name sequence)
    struct Ln { uint32_t seq; uint64_t before, after; };
    std::vector<Ln> lines;
    {
        const uint32_t ra = r.cpu_rank_index[index_of(rank_a)];
        const uint64_t a0 = h.line_off[ra], a1 = h.line_off[ra + 1];
        if (kind == 0) {
            for (uint64_t l = a0; l < a1; ++l) lines.push_back({uint32_t(h.lkey[l]), h.lcount[l], h.lcount[l]});
        } else {
            const uint32_t rb = r.cpu_rank_index[index_of(rank_b)];
            uint64_t i = a0, j = h.line_off[rb];
            const uint64_t b1 = h.line_off[rb + 1];
            while (i < a1 || j < b1) {
                const uint32_t si = i < a1 ? uint32_t(h.lkey[i]) : 0xffffffffu;
                const uint32_t sj = j < b1 ? uint32_t(h.lkey[j]) : 0xffffffffu;
                if (si == sj) lines.push_back({si, h.lcount[i++], h.lcount[j++]});
                else if (si < sj) lines.push_back({si, h.lcount[i++], 0});
                else lines.push_back({sj, 0, h.lcount[j++]});
            }
        }
    }
    // trie pre-order from the sorted lines
    std::vector<svg::Node> nodes;
    std::vector<size_t> open;  // node index per depth on the current path
    const uint32_t* prev = nullptr;
    uint64_t prev_len = 0, max_len = 0, tot_b = 0, tot_a = 0;
    for (const Ln& ln : lines) {
        const uint32_t g = h.dense_rep[ln.seq];
        const uint32_t* k = h.arena.data() + h.seq_off[g];
        const uint64_t len = h.seq_off[g + 1] - h.seq_off[g];
        uint64_t p = 0;
        while (p < len && p < prev_len && k[p] == prev[p]) ++p;
        open.resize(p);
        for (size_t d = 0; d < p; ++d) {
            nodes[open[d]].before += ln.before;
            nodes[open[d]].after += ln.after;
        }
        for (uint64_t d = p; d < len; ++d) {
            open.push_back(nodes.size());
            nodes.push_back({uint32_t(d), k[d], ln.before, ln.after});
        }
        tot_b += ln.before;
        tot_a += ln.after;
        max_len = std::max(max_len, len);
        prev = k;
        prev_len = len;
    }
    const bool diff = kind == 1;
    const int height = int(max_len + 2) * o.row_height + 24;
    std::ostringstream out;
    out << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << o.width << "\" height=\"" << height << "\">\n";
    out << "<rect width=\"100%\" height=\"100%\" fill=\"white\"/>\n";
    out << "<text x=\"8\" y=\"16\" font-size=\"13\" font-family=\"monospace\">" << svg::escape(o.title ? o.title : "")
        << "</text>\n";
    // per depth on the current path: x, width, the parent's count basis, the
    // next child's x, visible
    struct Lvl { double x, w, cx; uint64_t basis; bool vis; };
    std::vector<Lvl> lv;
    const Lvl root{0.0, double(o.width), 0.0, tot_a, true};
    for (const svg::Node& n : nodes) {
        lv.resize(n.depth);
        const Lvl& par = n.depth ? lv[n.depth - 1] : root;
        Lvl& pm = n.depth ? lv[n.depth - 1] : const_cast<Lvl&>(root);
        double w;
        if (n.depth == 0)
            w = tot_a ? double(o.width) * double(n.after) / double(tot_a) : 0.0;
        else
            w = par.basis ? par.w * double(n.after) / double(par.basis) : 0.0;
        const double x = pm.cx;
        pm.cx += w;
        const bool vis = par.vis && par.basis != 0 && w / o.width >= o.min_fraction && n.after > 0;
        lv.push_back({x, w, x, n.after, vis});
        if (!vis) continue;
        const std::string name = r.name_of(n.key);
        const int y = height - (int(n.depth) + 2) * o.row_height;
        out << "<g><title>" << svg::escape(name) << " (" << n.after;
        if (diff) out << " vs " << n.before;
        out << ")</title><rect x=\"" << x << "\" y=\"" << y << "\" width=\"" << w << "\" height=\""
            << o.row_height - 1 << "\" fill=\""
            << (diff ? svg::diff_color(n.before, n.after, tot_b, tot_a) : svg::name_color(name)) << "\"/>";
        if (w > 60)
            out << "<text x=\"" << x + 2 << "\" y=\"" << y + o.row_height - 4
                << "\" font-size=\"11\" font-family=\"monospace\">" << svg::escape(name) << "</text>";
        out << "</g>\n";
    }
    out << "</svg>\n";
    return out.str();
}
std::string groupdata_json(Ctx& c, uint32_t parts) {
    Result& r = *c.result;
    JsonW j;
    j.raw("{\"group\": ");
    j.num(r.group);
    j.raw(", \"cpu_profiles\": [");
    const bool cpu = parts & STG_GD_CPU;
    // bulk-copy what the lines need once
    std::vector<uint64_t> lk(cpu ? r.n_lines : 0), lc(cpu ? r.n_lines : 0), seq_off, line_off;
    std::vector<uint32_t> dense_rep(cpu ? r.n_seq : 0), arena;
    if (cpu && r.n_lines) {
        d2h(c, lk.data(), "lkey_s", r.n_lines);
        d2h(c, lc.data(), "lcount_s", r.n_lines);
        d2h(c, dense_rep.data(), "dense_rep", r.n_seq);
        size_t G = c.buf("seq_off").cap / sizeof(uint64_t);
        (void)G;
    }
    uint64_t G = 0;
    if (cpu && r.n_lines) {
        // number of gids = size of gids buffer in use; recover from seq_off's last entry
        G = r.n_gid;
        seq_off.resize(G + 1);
        d2h(c, seq_off.data(), "seq_off", G + 1);
        arena.resize(seq_off[G]);
        d2h(c, arena.data(), "arena", seq_off[G]);
        line_off.resize(r.n_window_ranks + 1);
        d2h(c, line_off.data(), "line_off", r.n_window_ranks + 1);
    }
    for (size_t i = 0; cpu && i < r.cpu_rank_ids.size(); ++i) {
        if (i) j.raw(", ");
        uint32_t row = r.cpu_rank_index[i];
        j.raw("{\"rank\": ");
        j.num(r.cpu_rank_ids[i]);
        j.raw(", \"total\": ");
        j.num(r.cpu_totals[i]);
        j.raw(", \"lines\": [");
        for (uint64_t l = line_off[row]; l < line_off[row + 1]; ++l) {
            if (l > line_off[row]) j.raw(", ");
            uint32_t g = dense_rep[uint32_t(lk[l])];
            j.raw("[[");
            for (uint64_t k = seq_off[g]; k < seq_off[g + 1]; ++k) {
                if (k > seq_off[g]) j.raw(", ");
                j.str(r.name_of(arena[k]));
            }
            j.raw("], ");
            j.num(lc[l]);
            j.raw("]");
        }
        j.raw("]}");
    }
    j.raw("], \"gpu_profiles\": [");
    bool first = true;
    for (const auto& [rank, m] : r.gpu) {
        if (!first) j.raw(", ");
        first = false;
        j.raw("{\"rank\": ");
        j.num(rank);
        j.raw(", \"kernels\": [");
        bool f2 = true;
        for (const auto& [k, v] : m) {
            if (!f2) j.raw(", ");
            f2 = false;
            j.raw("[");
            j.str(k);
            j.raw(", ");
            j.num(v);
            j.raw("]");
        }
        j.raw("]}");
    }
    j.raw("], \"os_snapshots\": [");
    first = true;
    for (const auto& [rank, a] : r.os) {
        if (!first) j.raw(", ");
        first = false;
        j.raw("{\"rank\": ");
        j.num(rank);
        for (int pass = 0; pass < 2; ++pass) {
            j.raw(pass ? ", \"softirqs\": [" : ", \"interrupts\": [");
            bool f2 = true;
            for (const auto& [k, v] : pass ? a.softirqs : a.interrupts) {
                if (!f2) j.raw(", ");
                f2 = false;
                j.raw("[");
                j.str(k);
                j.raw(", ");
                j.num(v);
                j.raw("]");
            }
            j.raw("]");
        }
        j.raw(", \"p50\": ");
        j.num(a.p50);
        j.raw(", \"p99\": ");
        j.num(a.p99);
        j.raw(", \"migrations\": ");
        j.num(a.migrations);
        j.raw("}");
    }
    j.raw("], \"lateness_per_instance\": [");
    if (r.n_windowed) {
        std::vector<double> lat(uint64_t(r.rank_span) * r.n_windowed);
        d2h(c, lat.data(), "lat", lat.size());
        for (uint64_t wi = 0; wi < r.n_windowed; ++wi) {
            if (wi) j.raw(", ");
            j.raw("[");
            bool f2 = true;
            for (int32_t rk = 0; rk < r.rank_span; ++rk) {
                double v = lat[uint64_t(rk) * r.n_windowed + wi];
                if (!(v == v)) continue;
                if (!f2) j.raw(", ");
                f2 = false;
                j.raw("[");
                j.num(rk);
                j.raw(", ");
                j.num(v);
                j.raw("]");
            }
            j.raw("]");
        }
    }
    j.raw("], \"iteration_times_ms\": [");
    for (size_t i = 0; i < r.iteration_times_ms.size(); ++i) {
        if (i) j.raw(", ");
        j.num(r.iteration_times_ms[i]);
    }
    j.raw("], \"baseline\": ");
    if (r.has_baseline) {
        j.raw("{\"delta\": ");
        j.num(r.baseline_delta);
        j.raw(", \"fractions\": [");
        bool f2 = true;
        for (const auto& [k, v] : r.baseline) {
            if (!f2) j.raw(", ");
            f2 = false;
            j.raw("[");
            j.str(k);
            j.raw(", ");
            j.num(v);
            j.raw("]");
        }
        j.raw("]}");
    } else {
        j.raw("null");
    }
    j.raw(", \"baseline_iteration_ms\": ");
    if (r.has_baseline_iteration)
        j.num(r.baseline_iteration_ms);
    else
        j.raw("null");
    j.raw("}");
    return j.s;
}

// compute_waterline / flag_ranks rendering from the device-resident result.
static std::string waterline_json_dist(Ctx& c) {
    Result& r = *c.result;
    const uint64_t NG = r.wl_NG, nf = r.wl_flags;
    std::vector<uint32_t> ukeys;  // global keys of the waterline's names (set in the byte map)
    {
        std::vector<uint8_t> um(r.wl_NGF);
        d2h(c, um.data(), "wl_umap", r.wl_NGF);
        for (uint64_t g = 0; g < r.wl_NGF; ++g)
            if (um[g]) ukeys.push_back(uint32_t(g));
    }
    std::vector<double> hm(NG), hs(NG);
    std::vector<unsigned> hnp(NG);
    d2h(c, hm.data(), "wlg_mean", NG);
    d2h(c, hs.data(), "wlg_sd", NG);
    d2h(c, hnp.data(), "wl_np", NG);
    std::vector<uint32_t> fr(nf), ff(nf);
    std::vector<double> ffr(nf), fth(nf);
    d2h(c, fr.data(), "wl_or", nf);
    d2h(c, ff.data(), "wl_of", nf);
    d2h(c, ffr.data(), "wl_ofr", nf);
    d2h(c, fth.data(), "wl_oth", nf);
    std::vector<int32_t> rids(r.n_window_ranks);
    d2h(c, rids.data(), "rids", r.n_window_ranks);
    std::vector<uint32_t> gkey(r.wl_F);  // dense name -> global key
    d2h(c, gkey.data(), "wl_gkey_g", r.wl_F);
    JsonW j;
    j.raw("{\"functions\": [");
    bool first = true;
    for (uint64_t g = 0; g < NG; ++g) {
        if (!hnp[g]) continue;
        if (!first) j.raw(", ");
        first = false;
        j.raw("[");
        j.str(r.gname(ukeys[g]));
        j.raw(", ");
        j.num(hm[g]);
        j.raw(", ");
        j.num(hs[g]);
        j.raw("]");
    }
    j.raw("], \"flags\": [");
    std::vector<size_t> order(nf);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        return fr[a] != fr[b] ? fr[a] < fr[b] : ff[a] < ff[b];
    });
    for (size_t i = 0; i < nf; ++i) {
        const size_t k = order[i];
        if (i) j.raw(", ");
        j.raw("[");
        j.num(int64_t(rids[fr[k]]));
        j.raw(", ");
        j.str(r.gname(gkey[ff[k]]));
        j.raw(", ");
        j.num(ffr[k]);
        j.raw(", ");
        j.num(fth[k]);
        j.raw("]");
    }
    j.raw("]}");
    r.waterline_json = j.s;
    return j.s;
}

std::string waterline_json(Ctx& c) {
    Result& r = *c.result;
    if (!r.waterline_json.empty()) return r.waterline_json;
    if (r.wl_dist) return waterline_json_dist(c);
    const uint64_t F = r.wl_F, nf = r.wl_flags;
    std::vector<double> hm(F), hs(F);
    std::vector<uint8_t> hp(F);
    std::vector<uint32_t> dense(F), fr(nf), ff(nf);
    std::vector<double> ffr(nf), fth(nf);
    d2h(c, hm.data(), "wl_mean", F);
    d2h(c, hs.data(), "wl_sd", F);
    d2h(c, hp.data(), "wl_pres", F);
    d2h(c, dense.data(), "dense_final", F);
    d2h(c, fr.data(), "wl_or", nf);
    d2h(c, ff.data(), "wl_of", nf);
    d2h(c, ffr.data(), "wl_ofr", nf);
    d2h(c, fth.data(), "wl_oth", nf);
    std::vector<int32_t> rids(r.n_window_ranks);
    d2h(c, rids.data(), "rids", r.n_window_ranks);
    JsonW j;
    j.raw("{\"functions\": [");
    bool first = true;
    for (uint64_t f = 0; f < F; ++f) {
        if (!hp[f]) continue;
        if (!first) j.raw(", ");
        first = false;
        j.raw("[");
        j.str(r.name_of(dense[f]));
        j.raw(", ");
        j.num(hm[f]);
        j.raw(", ");
        j.num(hs[f]);
        j.raw("]");
    }
    j.raw("], \"flags\": [");
    // flag_ranks order: ranks ascending, names in map order
    std::vector<size_t> order(nf);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        return fr[a] != fr[b] ? fr[a] < fr[b] : ff[a] < ff[b];
    });
    for (size_t i = 0; i < nf; ++i) {
        size_t k = order[i];
        if (i) j.raw(", ");
        j.raw("[");
        j.num(int64_t(rids[fr[k]]));
        j.raw(", ");
        j.str(r.name_of(dense[ff[k]]));
        j.raw(", ");
        j.num(ffr[k]);
        j.raw(", ");
        j.num(fth[k]);
        j.raw("]");
    }
    j.raw("]}");
    r.waterline_json = j.s;
    return j.s;
}

void window_run(Ctx& c, const stg_window& w, const stg_config& cfg) {
    if (!c.result) c.result = std::make_unique<Result>();
    Result& r = *c.result;
    r.render_valid = r.render_unk_ready = false;
    r.hf = Result::HostFold{};
    r.svg_key = ~0ull;
    Runner rn(c, w, cfg, r);
    rn.run();
}

}  // namespace stg
