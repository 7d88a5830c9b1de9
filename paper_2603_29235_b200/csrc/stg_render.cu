// stg_render.cu — device rendering of the folded-text artifacts that follow the
// hot path:
//
//   FoldedProfile::to_string   folded.cpp:33-43   "a;b;c <count>\n" per line
//   diff_folded(a, b)          folded.cpp:83-96   "a;b;c <count_a> <count_b>\n" over
//                                                 the union of both profiles' lines
//
// as written by `strata diagnose` (tools/strata.cpp:97-109, one diff per flagged
// rank against the reference rank) and `strata flamegraph` (:119-131).
//
// The window's folded profiles already live in HBM after stg_window_run: lines
// of every rank sorted by (rank, sequence rank) where the sequence rank is the
// byte-wise lexicographic position of the root-first name vector — exactly the
// std::map<std::vector<std::string>> order both reference functions iterate in.
// Rendering is therefore three byte-parallel passes over the lines:
//   1. line list: one rank's lines, or the sorted union of two ranks' lines
//      (radix sort of the concatenated sequence ranks + run heads);
//   2. per-line byte length (names + separators + decimal counts) and an
//      exclusive scan into text offsets;
//   3. one warp per line writes its bytes: a warp scan places the names, each
//      lane copies one name, lane 0 writes the counts.
// The names come from the dictionary blob the symbol tables' refresh left on the
// device (symtab.cu) and the window's unknown labels "[<build-id hex>+0x<off>]".
#include <cub/cub.cuh>

#include <cstring>

#include "result.h"
#include "stg_internal.h"

namespace stg {
namespace {

constexpr int kT = 256;
inline unsigned grid_of(uint64_t n, int per = kT) {
    uint64_t g = (n + per - 1) / per;
    return unsigned(g < 1 ? 1 : (g > 148ull * 64 ? 148ull * 64 : g));
}

struct Names {
    const uint64_t* dict_off;  // [n_dict + 1]
    const char* dict;
    const uint64_t* unk_final; // [n_unk] sorted final ranks of the unknown labels
    const uint64_t* unk_off;   // [n_unk + 1]
    const char* unk;
    uint32_t n_unk;
};

// Result::name_of on the device: unknown labels hold explicit final ranks, the
// dictionary fills the rest in order.
__device__ __forceinline__ void name_span(const Names& nm, uint32_t f, const char*& p, uint32_t& len) {
    uint32_t lo = 0, hi = nm.n_unk;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (nm.unk_final[mid] < f) lo = mid + 1; else hi = mid;
    }
    if (lo < nm.n_unk && nm.unk_final[lo] == f) {
        p = nm.unk + nm.unk_off[lo];
        len = uint32_t(nm.unk_off[lo + 1] - nm.unk_off[lo]);
    } else {
        const uint64_t d = uint64_t(f) - lo;
        p = nm.dict + nm.dict_off[d];
        len = uint32_t(nm.dict_off[d + 1] - nm.dict_off[d]);
    }
}

__device__ __forceinline__ uint32_t n_digits(unsigned long long v) {
    uint32_t n = 1;
    while (v >= 10) { v /= 10; ++n; }
    return n;
}

__device__ __forceinline__ void put_u64(char* o, unsigned long long v, uint32_t nd) {
    for (uint32_t k = nd; k-- > 0;) { o[k] = char('0' + v % 10); v /= 10; }
}

// Line list of one rank: sequence ranks and counts straight from the sorted lines.
__global__ void k_one_rank(uint64_t n, const uint64_t* lkey, const unsigned long long* lcnt, uint32_t* seq,
                           unsigned long long* ca) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        seq[i] = uint32_t(lkey[i]);
        ca[i] = lcnt[i];
    }
}

// Concatenation of two ranks' lines: key = sequence rank, value = side (bit 63)
// | line index.
__global__ void k_two_rank_keys(uint64_t na, uint64_t nb, const uint64_t* lkey_a, const uint64_t* lkey_b,
                                uint32_t* key, uint64_t* val) {
    const uint64_t n = na + nb;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        if (i < na) { key[i] = uint32_t(lkey_a[i]); val[i] = i; }
        else { key[i] = uint32_t(lkey_b[i - na]); val[i] = (1ull << 63) | (i - na); }
    }
}

__global__ void k_run_heads(uint64_t n, const uint32_t* key, uint32_t* head) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        head[i] = (i == 0 || key[i] != key[i - 1]) ? 1u : 0u;
}

// Each concatenated entry deposits its count on its side of output line
// scan[i] - 1 (a sequence occurs at most once per rank, so no two entries write
// the same cell).
__global__ void k_union_fill(uint64_t n, const uint32_t* key, const uint64_t* val, const uint32_t* scan,
                             const unsigned long long* lcnt_a, const unsigned long long* lcnt_b, uint32_t* seq,
                             unsigned long long* ca, unsigned long long* cb) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t o = scan[i] - 1;
        const uint64_t v = val[i];
        const bool side_b = v >> 63;
        const uint64_t l = v & ~(1ull << 63);
        if (i == 0 || key[i] != key[i - 1]) {
            seq[o] = key[i];
            // the partner (if any) is the next entry and writes the other side;
            // a lone entry zeroes it
            if (i + 1 == n || key[i + 1] != key[i]) {
                if (side_b) ca[o] = 0; else cb[o] = 0;
            }
        }
        if (side_b) cb[o] = lcnt_b[l]; else ca[o] = lcnt_a[l];
    }
}

struct Lines {
    const uint32_t* seq;                 // sequence rank per output line
    const unsigned long long* ca;
    const unsigned long long* cb;        // null: single-count lines (to_string)
    const uint32_t* dense_rep;           // sequence rank -> sequence id
    const uint64_t* seq_off;             // sequence id -> arena range
    const uint32_t* arena;               // final name ranks, root first
};

__global__ void k_line_bytes(uint64_t n, Lines L, Names nm, uint64_t* bytes) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t g = L.dense_rep[L.seq[i]];
        const uint64_t a0 = L.seq_off[g], a1 = L.seq_off[g + 1];
        uint64_t b = (a1 - a0) - 1 + 1 + n_digits(L.ca[i]) + 1;  // separators, ' ', count, '\n'
        if (L.cb) b += 1 + n_digits(L.cb[i]);
        for (uint64_t k = a0; k < a1; ++k) {
            const char* p;
            uint32_t len;
            name_span(nm, L.arena[k], p, len);
            b += len;
        }
        bytes[i] = b;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) bytes[n] = 0;
}

// One warp per line.  Names are placed 32 at a time with a warp scan of
// (length + 1); each lane copies its own name and the ';' after it.
__global__ void k_line_write(uint64_t n, Lines L, Names nm, const uint64_t* off, char* out) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n; i += nw) {
        const uint32_t g = L.dense_rep[L.seq[i]];
        const uint64_t a0 = L.seq_off[g], a1 = L.seq_off[g + 1];
        char* o = out + off[i];
        uint64_t pos = 0;
        for (uint64_t k0 = a0; k0 < a1; k0 += 32) {
            const uint64_t k = k0 + lane;
            const char* p = nullptr;
            uint32_t len = 0;
            if (k < a1) name_span(nm, L.arena[k], p, len);
            uint32_t w = k < a1 ? len + 1 : 0, incl = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += t;
            }
            if (k < a1) {
                char* q = o + pos + (incl - w);
                for (uint32_t c = 0; c < len; ++c) q[c] = p[c];
                q[len] = k + 1 < a1 ? ';' : ' ';
            }
            pos += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
            char* q = o + pos;
            const uint32_t da = n_digits(L.ca[i]);
            put_u64(q, L.ca[i], da);
            q += da;
            if (L.cb) {
                *q++ = ' ';
                const uint32_t db = n_digits(L.cb[i]);
                put_u64(q, L.cb[i], db);
                q += db;
            }
            *q = '\n';
        }
    }
}

template <class T>
T* dbuf(Ctx& c, const char* name, size_t n) { return c.buf(name).as<T>(n); }

template <class T>
T get1(Ctx& c, const T* d) {
    T v;
    STG_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    STG_CUDA(cudaStreamSynchronize(c.stream));
    return v;
}

// Upload the name blobs the arena's final ranks refer to.
Names stage_names(Ctx& c, Result& r) {
    // the dictionary blob is already on the device (symtab.cu, bufs dict_blob / dict_off)
    if (!r.render_unk_ready) {
        const size_t nu = r.unk_labels.size();
        std::vector<uint64_t> off(nu + 1, 0);
        for (size_t i = 0; i < nu; ++i) off[i + 1] = off[i] + r.unk_labels[i].size();
        std::string blob;
        for (const auto& s : r.unk_labels) blob += s;
        uint64_t* d_fin = dbuf<uint64_t>(c, "rd_unk_final", nu + 1);
        uint64_t* d_off = dbuf<uint64_t>(c, "rd_unk_off", nu + 1);
        char* d_blob = dbuf<char>(c, "rd_unk", blob.size() + 1);
        if (nu) STG_CUDA(cudaMemcpyAsync(d_fin, r.unk_final.data(), nu * 8, cudaMemcpyHostToDevice, c.stream));
        STG_CUDA(cudaMemcpyAsync(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice, c.stream));
        if (!blob.empty())
            STG_CUDA(cudaMemcpyAsync(d_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice, c.stream));
        STG_CUDA(cudaStreamSynchronize(c.stream));
        r.render_unk_ready = true;
    }
    return Names{static_cast<const uint64_t*>(c.buf("dict_off").p), static_cast<const char*>(c.buf("dict_blob").p),
                 static_cast<const uint64_t*>(c.buf("rd_unk_final").p),
                 static_cast<const uint64_t*>(c.buf("rd_unk_off").p), static_cast<const char*>(c.buf("rd_unk").p),
                 uint32_t(r.unk_labels.size())};
}

// rank id -> row of the window's sorted lines; the reference's rank_profile
// error (tools/strata.cpp:111-116) when the rank has no profile.
uint32_t profile_row(Ctx& c, Result& r, int32_t rank) {
    auto it = std::lower_bound(r.cpu_rank_ids.begin(), r.cpu_rank_ids.end(), rank);
    if (it == r.cpu_rank_ids.end() || *it != rank) {
        if (c.world > 1) fail(STG_EINVAL, "rank " + std::to_string(rank) + " has no profile on this context");
        fail(STG_EINVAL, "unknown rank id: " + std::to_string(rank));
    }
    return r.cpu_rank_index[size_t(it - r.cpu_rank_ids.begin())];
}

}  // namespace

// Render into the device buffer "rd_text"; returns the byte count (no NUL).
uint64_t render_folded(Ctx& c, int kind, int32_t rank_a, int32_t rank_b) {
    Result& r = *c.result;
    if (r.render_valid && r.render_kind == kind && r.render_a == rank_a && r.render_b == rank_b)
        return r.render_len;
    r.render_valid = false;
    const uint32_t row_a = profile_row(c, r, rank_a);
    const uint32_t row_b = kind == 1 ? profile_row(c, r, rank_b) : 0;
    cudaStream_t st = c.stream;
    const uint64_t* line_off = static_cast<const uint64_t*>(c.buf("line_off").p);
    const uint64_t* lkey = static_cast<const uint64_t*>(c.buf("lkey_s").p);
    const auto* lcnt = static_cast<const unsigned long long*>(c.buf("lcount_s").p);
    uint64_t ra[2], rb[2] = {0, 0};
    STG_CUDA(cudaMemcpyAsync(ra, line_off + row_a, 16, cudaMemcpyDeviceToHost, st));
    if (kind == 1) STG_CUDA(cudaMemcpyAsync(rb, line_off + row_b, 16, cudaMemcpyDeviceToHost, st));
    STG_CUDA(cudaStreamSynchronize(st));
    const uint64_t na = ra[1] - ra[0], nb = rb[1] - rb[0];
    uint64_t n;
    uint32_t* seq;
    unsigned long long *ca, *cb = nullptr;
    if (kind == 0) {
        n = na;
        seq = dbuf<uint32_t>(c, "rd_seq", n);
        ca = dbuf<unsigned long long>(c, "rd_ca", n);
        if (n) k_one_rank<<<grid_of(n), kT, 0, st>>>(n, lkey + ra[0], lcnt + ra[0], seq, ca);
    } else {
        const uint64_t m = na + nb;
        uint32_t* key = dbuf<uint32_t>(c, "rd_key", m);
        uint64_t* val = dbuf<uint64_t>(c, "rd_val", m);
        uint32_t* key_s = dbuf<uint32_t>(c, "rd_key_s", m);
        uint64_t* val_s = dbuf<uint64_t>(c, "rd_val_s", m);
        uint32_t* head = dbuf<uint32_t>(c, "rd_head", m);
        uint32_t* scan = dbuf<uint32_t>(c, "rd_scan", m);
        seq = dbuf<uint32_t>(c, "rd_seq", m);
        ca = dbuf<unsigned long long>(c, "rd_ca", m);
        cb = dbuf<unsigned long long>(c, "rd_cb", m);
        n = 0;
        if (m) {
            k_two_rank_keys<<<grid_of(m), kT, 0, st>>>(na, nb, lkey + ra[0], lkey + rb[0], key, val);
            size_t tb = 0;
            STG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key_s, val, val_s, int64_t(m), 0, 32, st));
            void* tmp = c.buf("rd_tmp").get(tb);
            STG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key_s, val, val_s, int64_t(m), 0, 32, st));
            k_run_heads<<<grid_of(m), kT, 0, st>>>(m, key_s, head);
            tb = 0;
            STG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, head, scan, int64_t(m), st));
            tmp = c.buf("rd_tmp").get(tb);
            STG_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, head, scan, int64_t(m), st));
            k_union_fill<<<grid_of(m), kT, 0, st>>>(m, key_s, val_s, scan, lcnt + ra[0], lcnt + rb[0], seq, ca, cb);
            n = get1(c, scan + m - 1);
        }
    }
    STG_CUDA(cudaGetLastError());
    uint64_t total = 0;
    if (n) {
        const Names nm = stage_names(c, r);
        const Lines L{seq, ca, cb, static_cast<const uint32_t*>(c.buf("dense_rep").p),
                      static_cast<const uint64_t*>(c.buf("seq_off").p),
                      static_cast<const uint32_t*>(c.buf("arena").p)};
        uint64_t* bytes = dbuf<uint64_t>(c, "rd_bytes", n + 1);
        uint64_t* off = dbuf<uint64_t>(c, "rd_off", n + 1);
        k_line_bytes<<<grid_of(n), kT, 0, st>>>(n, L, nm, bytes);
        size_t tb = 0;
        STG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, bytes, off, int64_t(n + 1), st));
        void* tmp = c.buf("rd_tmp").get(tb);
        STG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, bytes, off, int64_t(n + 1), st));
        total = get1(c, off + n);
        char* text = dbuf<char>(c, "rd_text", total + 1);
        k_line_write<<<grid_of(n * 32), kT, 0, st>>>(n, L, nm, off, text);
        STG_CUDA(cudaGetLastError());
        STG_CUDA(cudaStreamSynchronize(st));
    }
    r.render_valid = true;
    r.render_kind = kind;
    r.render_a = rank_a;
    r.render_b = rank_b;
    r.render_len = total;
    return total;
}

// Copy the rendered text (plus NUL) into a host buffer of cap bytes.
void render_copy(Ctx& c, char* buf, uint64_t len) {
    if (len) {
        STG_CUDA(cudaMemcpyAsync(buf, c.buf("rd_text").p, len, cudaMemcpyDeviceToHost, c.stream));
        STG_CUDA(cudaStreamSynchronize(c.stream));
    }
    buf[len] = '\0';
}

}  // namespace stg
