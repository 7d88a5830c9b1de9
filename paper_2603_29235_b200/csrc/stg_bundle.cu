// stg_bundle.cu — bundle ingest on the GPU:
// load_bundle (proj/core/src/bundle.cpp:181-233) for the two bulk files,
//
//   samples.jsonl      one StackSample per line (sample_from_json, :44-56):
//                      {"frames":[["<40 hex>",offset],...],"rank":R,"spaces":"..","thread":T,"ts":N}
//   collectives.jsonl  one CollectiveEvent per line (:206-215):
//                      {"entry":N,"exit":N,"gpu_duration":N,"group":G,"kind":"AllReduce","rank":R}
//
// decoded straight into the stg_window SoA in HBM.  The file bytes are copied
// in once; then
//   1. line index      newline positions by flag + select (empty lines skipped,
//                      as std::getline + `if (line.empty()) continue`)
//   2. k_samples_a     thread per line: a JSON parser for one line (objects in
//                      any key order, nested skipping, integer values), rank /
//                      ts / frame count, build ids (BuildId::from_hex, :107-116)
//                      interned into a small device table
//   3. stable radix sort of the lines by rank (LoadedBundle::samples is a
//      std::map<int, vector>: ranks ascending, file order within a rank),
//      run-length encode -> rank_ids / rank_sample_off, scan -> frame offsets
//   4. k_samples_b     thread per sample: parse its line again, write frames
//   5. k_colls         thread per line of collectives.jsonl, file order kept.
// Errors: the first bad line in file order wins; build-id and collective-kind
// errors carry the reference's messages ("build id hex must be 40 chars",
// "build id hex has non-hex character", "unknown collective kind: X"); malformed
// JSON reports "<file> line N: <what>" (nlohmann's parse_error text is not
// reproduced).  Numbers must be integers (the writer, bundle.cpp:31-42, only
// emits integers for these fields).
#include <cub/cub.cuh>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "bundle.h"
#include "stg_internal.h"

namespace stg {
namespace {

constexpr int kT = 256;
inline unsigned grid_of(uint64_t n) {
    uint64_t g = (n + kT - 1) / kT;
    return unsigned(g < 1 ? 1 : (g > 148ull * 64 ? 148ull * 64 : g));
}

enum : uint32_t {
    E_OK = 0,
    E_SYNTAX = 1,     // malformed JSON
    E_MISSING = 2,    // required key absent
    E_TYPE = 3,       // value of the wrong JSON type
    E_HEXLEN = 4,     // build id hex must be 40 chars
    E_HEXCHAR = 5,    // build id hex has non-hex character
    E_NUMBER = 6,     // non-integer or out-of-range number
    E_BINS = 7,       // too many distinct build ids
    E_KIND = 8,       // unknown collective kind
};

// ------------------------------------------------------------ one-line parser
struct Cur {
    const uint8_t* p;
    uint64_t i, e;
    uint32_t err;
    __device__ uint32_t peek() const { return i < e ? p[i] : 0x100u; }
    __device__ void ws() {
        while (i < e && (p[i] == ' ' || p[i] == '\t' || p[i] == '\r' || p[i] == '\n')) ++i;
    }
    __device__ bool eat(uint8_t c) {
        ws();
        if (peek() == c) { ++i; return true; }
        return false;
    }
    __device__ void bad(uint32_t code) {
        if (!err) err = code;
    }
    // string -> raw content range [s0, s1); false on syntax error
    __device__ bool str(uint64_t& s0, uint64_t& s1, bool& esc) {
        ws();
        if (peek() != '"') { bad(E_TYPE); return false; }
        s0 = ++i;
        esc = false;
        while (i < e && p[i] != '"') {
            if (p[i] == '\\') { esc = true; ++i; }
            ++i;
        }
        if (i >= e) { bad(E_SYNTAX); return false; }
        s1 = i++;
        return true;
    }
    // integer; neg allowed if sgn
    __device__ bool integer(unsigned long long& v, bool& neg) {
        ws();
        neg = false;
        if (peek() == '-') { neg = true; ++i; }
        const uint32_t c0 = peek();
        if (c0 == '"' || c0 == '[' || c0 == '{' || c0 == 't' || c0 == 'f' || c0 == 'n') { bad(E_TYPE); return false; }
        if (c0 < '0' || c0 > '9') { bad(E_SYNTAX); return false; }
        v = 0;
        while (i < e && p[i] >= '0' && p[i] <= '9') {
            const unsigned d = p[i] - '0';
            if (v > (~0ull - d) / 10) { bad(E_NUMBER); return false; }
            v = v * 10 + d;
            ++i;
        }
        const uint32_t c = peek();
        if (c == '.' || c == 'e' || c == 'E') { bad(E_NUMBER); return false; }
        return true;
    }
    __device__ bool i64(long long& out) {
        unsigned long long v;
        bool neg;
        if (!integer(v, neg)) return false;
        if ((!neg && v > 0x7fffffffffffffffull) || (neg && v > 0x8000000000000000ull)) { bad(E_NUMBER); return false; }
        out = neg ? (long long)(0 - v) : (long long)v;
        return true;
    }
    __device__ bool u64(unsigned long long& out) {
        bool neg;
        if (!integer(out, neg)) return false;
        if (neg && out) { bad(E_NUMBER); return false; }  // get<uint64_t> of a negative number
        return true;
    }
    // any JSON value
    __device__ bool skip() {
        ws();
        const uint32_t c = peek();
        if (c == '"') {
            uint64_t a, b;
            bool x;
            return str(a, b, x);
        }
        if (c == '{' || c == '[') {
            int depth = 0;
            while (i < e) {
                const uint8_t ch = p[i];
                if (ch == '"') {
                    uint64_t a, b;
                    bool x;
                    if (!str(a, b, x)) return false;
                    continue;
                }
                ++i;
                if (ch == '{' || ch == '[') ++depth;
                else if (ch == '}' || ch == ']') {
                    if (--depth == 0) return true;
                }
            }
            bad(E_SYNTAX);
            return false;
        }
        if (c == 't' || c == 'f' || c == 'n' || c == '-' || (c >= '0' && c <= '9')) {
            while (i < e && p[i] != ',' && p[i] != '}' && p[i] != ']' && p[i] != ' ' && p[i] != '\t' &&
                   p[i] != '\r' && p[i] != '\n')
                ++i;
            return true;
        }
        bad(E_SYNTAX);
        return false;
    }
    __device__ bool key_is(uint64_t s0, uint64_t s1, const char* k) const {
        uint64_t n = 0;
        while (k[n]) ++n;
        if (s1 - s0 != n) return false;
        for (uint64_t j = 0; j < n; ++j)
            if (p[s0 + j] != uint8_t(k[j])) return false;
        return true;
    }
    // after a value inside an object: ',' -> true (more), '}' -> false (done)
    __device__ bool next_member(bool& more) {
        ws();
        if (peek() == ',') { ++i; more = true; return true; }
        if (peek() == '}') { ++i; more = false; return true; }
        bad(E_SYNTAX);
        return false;
    }
    __device__ bool end_of_line() {
        ws();
        if (i != e) { bad(E_SYNTAX); return false; }
        return true;
    }
};

__device__ __forceinline__ int hexv(uint8_t c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
}

// Build-id table: slot = {3 x u64 key (20 id bytes, zero padded), state}.
constexpr uint32_t kIdCap = 1024;  // power of two; at most kIdCap / 2 binaries
struct IdSlot {
    unsigned long long k0, k1, k2;
    unsigned int state;  // 0 empty, 1 writing, 2 ready
    unsigned int pad;
};

__device__ uint32_t id_get(IdSlot* T, const unsigned long long k[3], unsigned* used, uint32_t* err) {
    uint32_t h = uint32_t((k[0] * 0x9e3779b97f4a7c15ull) >> 40) & (kIdCap - 1);
    for (uint32_t probe = 0; probe < kIdCap; ++probe) {
        volatile IdSlot* s = T + h;
        unsigned st = s->state;
        if (st == 0) {
            if (atomicCAS(&T[h].state, 0u, 1u) == 0u) {
                s->k0 = k[0];
                s->k1 = k[1];
                s->k2 = k[2];
                __threadfence();
                atomicExch(&T[h].state, 2u);
                if (atomicAdd(used, 1u) + 1 > kIdCap / 2) *err = E_BINS;
                return h;
            }
            st = s->state;
        }
        while (st == 1) st = s->state;
        __threadfence();
        if (s->k0 == k[0] && s->k1 == k[1] && s->k2 == k[2]) return h;
        h = (h + 1) & (kIdCap - 1);
    }
    *err = E_BINS;
    return 0;
}

__device__ bool hex_id(Cur& c, uint64_t s0, uint64_t s1, bool esc, unsigned long long k[3]) {
    if (esc) { c.bad(E_SYNTAX); return false; }  // escaped hex is not produced by the writer
    if (s1 - s0 != 40) { c.bad(E_HEXLEN); return false; }
    k[0] = k[1] = k[2] = 0;
    for (int j = 0; j < 20; ++j) {
        const int hi = hexv(c.p[s0 + 2 * j]), lo = hexv(c.p[s0 + 2 * j + 1]);
        if (hi < 0 || lo < 0) { c.bad(E_HEXCHAR); return false; }
        k[j >> 3] |= uint64_t(hi << 4 | lo) << (8 * (j & 7));
    }
    return true;
}

struct LineOut {
    long long ts;
    unsigned long long frames_at;  // byte offset of the (last) "frames" value
    int rank;
    uint32_t n_frames;
    uint32_t err;
    uint32_t pad;
};

// Pass A over one samples.jsonl line.
__device__ void sample_line_a(const uint8_t* p, uint64_t s, uint64_t e, IdSlot* T, unsigned* used, uint32_t* terr,
                              LineOut& o) {
    Cur c{p, s, e, 0};
    o = LineOut{0, 0, 0, 0, 0, 0};
    bool has_f = false, has_r = false, has_t = false, has_ts = false, has_sp = false;
    if (!c.eat('{')) { c.bad(E_SYNTAX); o.err = c.err; return; }
    c.ws();
    bool more = c.peek() != '}';
    if (!more) ++c.i;
    while (more && !c.err) {
        uint64_t k0, k1;
        bool kesc;
        if (!c.str(k0, k1, kesc)) { c.err = c.err == E_TYPE ? E_SYNTAX : c.err; break; }
        if (!c.eat(':')) { c.bad(E_SYNTAX); break; }
        if (c.key_is(k0, k1, "frames")) {
            c.ws();
            o.frames_at = c.i;
            has_f = true;
            if (!c.eat('[')) { c.bad(E_TYPE); break; }
            uint32_t nf = 0;
            c.ws();
            bool fm = c.peek() != ']';
            if (!fm) ++c.i;
            while (fm && !c.err) {
                if (!c.eat('[')) { c.bad(E_TYPE); break; }
                uint64_t h0, h1;
                bool hesc;
                if (!c.str(h0, h1, hesc)) break;
                unsigned long long key[3];
                if (!hex_id(c, h0, h1, hesc, key)) break;
                if (!c.eat(',')) { c.bad(E_SYNTAX); break; }
                unsigned long long off;
                if (!c.u64(off)) break;
                if (!c.eat(']')) { c.bad(E_SYNTAX); break; }
                id_get(T, key, used, terr);
                ++nf;
                c.ws();
                if (c.peek() == ',') { ++c.i; }
                else if (c.peek() == ']') { ++c.i; fm = false; }
                else c.bad(E_SYNTAX);
            }
            o.n_frames = nf;
        } else if (c.key_is(k0, k1, "rank")) {
            long long v;
            if (!c.i64(v)) break;
            o.rank = int(v);
            has_r = true;
        } else if (c.key_is(k0, k1, "ts")) {
            long long v;
            if (!c.i64(v)) break;
            o.ts = v;
            has_ts = true;
        } else if (c.key_is(k0, k1, "thread")) {
            long long v;
            if (!c.i64(v)) break;
            has_t = true;
        } else if (c.key_is(k0, k1, "spaces")) {
            uint64_t a, b;
            bool x;
            if (!c.str(a, b, x)) break;
            has_sp = true;
        } else if (!c.skip()) {
            break;
        }
        if (!c.next_member(more)) break;
    }
    if (!c.err) c.end_of_line();
    // sample_from_json reads ts, rank, thread, frames, spaces in that order (:46-55)
    if (!c.err && (!has_ts || !has_r || !has_t || !has_f || !has_sp)) c.err = E_MISSING;
    o.err = c.err;
}

__global__ void k_line_bounds(uint64_t n_nl, const unsigned long long* nl, uint64_t size, uint64_t* ls,
                              uint64_t* le) {
    // line j = (nl[j-1] + 1, nl[j]); the last line ends at the file end
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j <= n_nl; j += uint64_t(gridDim.x) * blockDim.x) {
        ls[j] = j == 0 ? 0 : nl[j - 1] + 1;
        le[j] = j < n_nl ? nl[j] : size;
    }
}

struct NlFlag {
    const uint8_t* p;
    __device__ bool operator()(const unsigned long long& i) const { return p[i] == '\n'; }
};
struct NonEmpty {
    const uint64_t* ls;
    const uint64_t* le;
    __device__ bool operator()(const uint32_t& j) const { return le[j] > ls[j]; }
};

__global__ void k_samples_a(const uint8_t* p, uint64_t nl, const uint32_t* lines, const uint64_t* ls,
                            const uint64_t* le, IdSlot* T, unsigned* used, uint32_t* terr, LineOut* out,
                            unsigned long long* first_err, int* key) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < nl; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t L = lines[j];
        LineOut o;
        sample_line_a(p, ls[L], le[L], T, used, terr, o);
        out[j] = o;
        key[j] = o.rank;
        if (o.err) atomicMin(first_err, (unsigned long long)j);
    }
}

// bin of every id slot: compacted order of the used slots
__global__ void k_id_compact(const IdSlot* T, uint32_t* bin_of, uint8_t* ids, unsigned* n) {
    if (blockIdx.x || threadIdx.x) return;
    unsigned b = 0;
    for (uint32_t h = 0; h < kIdCap; ++h) {
        if (T[h].state == 2) {
            bin_of[h] = b;
            const unsigned long long k[3] = {T[h].k0, T[h].k1, T[h].k2};
            for (int j = 0; j < 20; ++j) ids[20 * b + j] = uint8_t(k[j >> 3] >> (8 * (j & 7)));
            ++b;
        }
    }
    *n = b;
}

__global__ void k_samples_b(const uint8_t* p, uint64_t ns, const uint32_t* order, const uint32_t* lines,
                            const uint64_t* le, const LineOut* out, const uint64_t* foff, const IdSlot* T,
                            const uint32_t* bin_of, int64_t* ts, uint64_t* pc, uint16_t* bin) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < ns; k += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t j = order[k];
        const LineOut& o = out[j];
        ts[k] = o.ts;
        Cur c{p, o.frames_at, le[lines[j]], 0};
        uint64_t f = foff[k];
        c.eat('[');
        for (uint32_t n = 0; n < o.n_frames; ++n) {
            c.eat('[');
            uint64_t h0, h1;
            bool esc;
            c.str(h0, h1, esc);
            unsigned long long key[3];
            hex_id(c, h0, h1, esc, key);
            c.eat(',');
            unsigned long long off;
            c.u64(off);
            c.eat(']');
            c.eat(',');
            uint32_t h = uint32_t((key[0] * 0x9e3779b97f4a7c15ull) >> 40) & (kIdCap - 1);
            while (!(T[h].k0 == key[0] && T[h].k1 == key[1] && T[h].k2 == key[2] && T[h].state == 2))
                h = (h + 1) & (kIdCap - 1);
            pc[f] = off;
            bin[f] = uint16_t(bin_of[h]);
            ++f;
        }
    }
}

struct CollOut {
    uint32_t err;
    uint32_t kind_s0_rel, kind_len;  // for the "unknown collective kind" message
    uint32_t pad;
};

__device__ bool bytes_eq(const uint8_t* p, uint64_t s0, uint64_t s1, const char* k) {
    uint64_t n = 0;
    while (k[n]) ++n;
    if (s1 - s0 != n) return false;
    for (uint64_t j = 0; j < n; ++j)
        if (p[s0 + j] != uint8_t(k[j])) return false;
    return true;
}

__global__ void k_colls(const uint8_t* p, uint64_t nl, const uint32_t* lines, const uint64_t* ls, const uint64_t* le,
                        int32_t* rank, int32_t* group, uint8_t* kind, int64_t* entry, int64_t* exit_,
                        int64_t* dur, CollOut* cout, unsigned long long* first_err) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < nl; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t L = lines[j];
        Cur c{p, ls[L], le[L], 0};
        CollOut o{0, 0, 0, 0};
        bool h_r = false, h_g = false, h_k = false, h_en = false, h_ex = false, h_d = false;
        long long vr = 0, vg = 0, ven = 0, vex = 0, vd = 0;
        uint64_t ks0 = 0, ks1 = 0;
        if (!c.eat('{')) c.bad(E_SYNTAX);
        c.ws();
        bool more = !c.err && c.peek() != '}';
        if (!c.err && !more) ++c.i;
        while (more && !c.err) {
            uint64_t k0, k1;
            bool kesc;
            if (!c.str(k0, k1, kesc)) { c.err = E_SYNTAX; break; }
            if (!c.eat(':')) { c.bad(E_SYNTAX); break; }
            if (c.key_is(k0, k1, "rank")) { if (!c.i64(vr)) break; h_r = true; }
            else if (c.key_is(k0, k1, "group")) { if (!c.i64(vg)) break; h_g = true; }
            else if (c.key_is(k0, k1, "entry")) { if (!c.i64(ven)) break; h_en = true; }
            else if (c.key_is(k0, k1, "exit")) { if (!c.i64(vex)) break; h_ex = true; }
            else if (c.key_is(k0, k1, "gpu_duration")) { if (!c.i64(vd)) break; h_d = true; }
            else if (c.key_is(k0, k1, "kind")) {
                bool esc;
                if (!c.str(ks0, ks1, esc)) break;
                h_k = true;
            } else if (!c.skip()) break;
            if (!c.next_member(more)) break;
        }
        if (!c.err) c.end_of_line();
        if (!c.err && (!h_r || !h_g || !h_k || !h_en || !h_ex || !h_d)) c.err = E_MISSING;
        uint8_t kd = 0;
        if (!c.err) {
            if (bytes_eq(p, ks0, ks1, "AllReduce")) kd = 0;
            else if (bytes_eq(p, ks0, ks1, "ReduceScatter")) kd = 1;
            else if (bytes_eq(p, ks0, ks1, "AllGather")) kd = 2;
            else if (bytes_eq(p, ks0, ks1, "Broadcast")) kd = 3;
            else if (bytes_eq(p, ks0, ks1, "P2P")) kd = 4;
            else {
                c.err = E_KIND;
                o.kind_s0_rel = uint32_t(ks0 - ls[L]);
                o.kind_len = uint32_t(ks1 - ks0);
            }
        }
        o.err = c.err;
        cout[j] = o;
        if (c.err) atomicMin(first_err, (unsigned long long)j);
        rank[j] = int32_t(vr);
        group[j] = int32_t(vg);
        kind[j] = kd;
        entry[j] = ven;
        exit_[j] = vex;
        dur[j] = vd;
    }
}

__global__ void k_iota_u32(uint64_t n, uint32_t* v) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        v[i] = uint32_t(i);
}

__global__ void k_sorted_nf(uint64_t n, const uint32_t* ord, const LineOut* out, uint64_t* nf) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k <= n; k += uint64_t(gridDim.x) * blockDim.x)
        nf[k] = k < n ? out[ord[k]].n_frames : 0;
}

const char* what(uint32_t code) {
    switch (code) {
        case E_SYNTAX: return "malformed JSON";
        case E_MISSING: return "missing key";
        case E_TYPE: return "value of the wrong type";
        case E_NUMBER: return "number is not an integer in range";
        case E_BINS: return "more than 512 distinct build ids";
        default: return "invalid record";
    }
}

template <class T>
T* dbuf(Ctx& c, const std::string& name, size_t n) { return c.buf(name).as<T>(n); }

template <class T>
T get1(Ctx& c, const T* d) {
    T v;
    STG_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    STG_CUDA(cudaStreamSynchronize(c.stream));
    return v;
}

// Newline-delimited non-empty lines of the device bytes -> (ls, le) and the
// index list of non-empty lines.  Returns the number of non-empty lines.
uint64_t index_lines(Ctx& c, const std::string& tag, const uint8_t* d, uint64_t size, const uint64_t*& ls,
                     const uint64_t*& le, const uint32_t*& lines, uint64_t& n_all) {
    cudaStream_t st = c.stream;
    unsigned long long* nl = dbuf<unsigned long long>(c, tag + "_nl", size + 1);
    unsigned long long* nnl = dbuf<unsigned long long>(c, tag + "_nnl", 1);
    size_t tb = 0;
    cub::CountingInputIterator<unsigned long long> it(0);
    STG_CUDA(cub::DeviceSelect::If(nullptr, tb, it, nl, nnl, int64_t(size), NlFlag{d}, st));
    STG_CUDA(cub::DeviceSelect::If(c.buf("bd_tmp").get(tb), tb, it, nl, nnl, int64_t(size), NlFlag{d}, st));
    const uint64_t n_nl = size ? get1(c, nnl) : 0;
    n_all = n_nl + 1;
    uint64_t* d_ls = dbuf<uint64_t>(c, tag + "_ls", n_all);
    uint64_t* d_le = dbuf<uint64_t>(c, tag + "_le", n_all);
    k_line_bounds<<<grid_of(n_all), kT, 0, st>>>(n_nl, nl, size, d_ls, d_le);
    uint32_t* idx = dbuf<uint32_t>(c, tag + "_lines", n_all);
    unsigned long long* nsel = dbuf<unsigned long long>(c, tag + "_nsel", 1);
    cub::CountingInputIterator<uint32_t> it2(0);
    tb = 0;
    STG_CUDA(cub::DeviceSelect::If(nullptr, tb, it2, idx, nsel, int64_t(n_all), NonEmpty{d_ls, d_le}, st));
    STG_CUDA(cub::DeviceSelect::If(c.buf("bd_tmp").get(tb), tb, it2, idx, nsel, int64_t(n_all),
                                   NonEmpty{d_ls, d_le}, st));
    ls = d_ls;
    le = d_le;
    lines = idx;
    return get1(c, nsel);
}

}  // namespace

// The file is read with pread(2) by kUpThreads threads, chunk j by thread
// j % kUpThreads, each into its own pair of pinned staging buffers and copied to
// the device on its own stream while its next chunk is read (page-cache reads
// of one thread top out near 7 GB/s).
constexpr int kUpThreads = 4;
constexpr size_t kChunk = 16u << 20;

const uint8_t* upload_file(Ctx& c, const std::string& path, const std::string& tag, uint64_t& size) {
    const int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) fail(STG_EINVAL, "missing bundle file: " + path);
    struct stat sb;
    if (fstat(fd, &sb) != 0) {
        ::close(fd);
        fail(STG_EINVAL, "cannot stat " + path);
    }
    size = uint64_t(sb.st_size);
    uint8_t* d = dbuf<uint8_t>(c, tag + "_bytes", size + 1);
    if (c.up.empty()) {
        c.up.resize(kUpThreads);
        for (auto& u : c.up) {
            STG_CUDA(cudaStreamCreateWithFlags(&u.stream, cudaStreamNonBlocking));
            for (int k = 0; k < 2; ++k) {
                STG_CUDA(cudaHostAlloc(&u.pin[k], kChunk, cudaHostAllocDefault));
                STG_CUDA(cudaEventCreateWithFlags(&u.ev[k], cudaEventDisableTiming));
            }
        }
    }
    const uint64_t n_chunks = (size + kChunk - 1) / kChunk;
    std::vector<std::string> errs(kUpThreads);
    auto work = [&](int t) {
        Ctx::Uploader& u = c.up[size_t(t)];
        int k = 0;
        for (uint64_t j = uint64_t(t); j < n_chunks; j += kUpThreads) {
            if (cudaEventSynchronize(u.ev[k]) != cudaSuccess) { errs[size_t(t)] = "cuda event"; return; }
            const uint64_t off = j * kChunk;
            const size_t want = size_t(std::min<uint64_t>(kChunk, size - off));
            size_t got = 0;
            while (got < want) {
                const ssize_t r = ::pread(fd, static_cast<uint8_t*>(u.pin[k]) + got, want - got, off_t(off + got));
                if (r <= 0) { errs[size_t(t)] = "short read of " + path; return; }
                got += size_t(r);
            }
            if (cudaMemcpyAsync(d + off, u.pin[k], want, cudaMemcpyHostToDevice, u.stream) != cudaSuccess ||
                cudaEventRecord(u.ev[k], u.stream) != cudaSuccess) {
                errs[size_t(t)] = "cuda copy";
                return;
            }
            k ^= 1;
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < kUpThreads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    ::close(fd);
    for (const auto& e : errs)
        if (!e.empty()) fail(STG_EINVAL, e);
    for (auto& u : c.up) STG_CUDA(cudaStreamSynchronize(u.stream));
    return d;
}

void bundle_decode_samples(Ctx& c, const uint8_t* d, uint64_t size, BundleBulk& b) {
    cudaStream_t st = c.stream;
    const uint64_t *ls, *le;
    const uint32_t* lines;
    uint64_t n_all;
    const uint64_t nl = index_lines(c, "bs", d, size, ls, le, lines, n_all);
    if (nl >= (1ull << 32)) fail(STG_EINVAL, "samples.jsonl: more than 2^32 - 1 samples");
    IdSlot* T = dbuf<IdSlot>(c, "bs_ids", kIdCap);
    unsigned* used = dbuf<unsigned>(c, "bs_used", 2);
    STG_CUDA(cudaMemsetAsync(T, 0, kIdCap * sizeof(IdSlot), st));
    STG_CUDA(cudaMemsetAsync(used, 0, 8, st));
    LineOut* out = dbuf<LineOut>(c, "bs_out", nl);
    int* key = dbuf<int>(c, "bs_key", nl);
    unsigned long long* ferr = dbuf<unsigned long long>(c, "bs_err", 1);
    STG_CUDA(cudaMemsetAsync(ferr, 0xff, 8, st));
    if (nl) k_samples_a<<<grid_of(nl), kT, 0, st>>>(d, nl, lines, ls, le, T, used, used + 1, out, ferr, key);
    STG_CUDA(cudaGetLastError());
    const unsigned long long e = get1(c, ferr);
    if (e != ~0ull) {
        LineOut o;
        uint32_t L;
        STG_CUDA(cudaMemcpyAsync(&o, out + e, sizeof o, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaMemcpyAsync(&L, lines + e, 4, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
        if (o.err == E_HEXLEN) fail(STG_EINVAL, "build id hex must be 40 chars");
        if (o.err == E_HEXCHAR) fail(STG_EINVAL, "build id hex has non-hex character");
        fail(STG_EINVAL, "samples.jsonl line " + std::to_string(L + 1) + ": " + what(o.err));
    }
    if (get1(c, used + 1)) fail(STG_EINVAL, std::string("samples.jsonl: ") + what(E_BINS));
    // build ids -> bins
    uint32_t* bin_of = dbuf<uint32_t>(c, "bs_bin_of", kIdCap);
    uint8_t* ids = dbuf<uint8_t>(c, "bs_idbytes", kIdCap * 20);
    unsigned* nbins = dbuf<unsigned>(c, "bs_nbins", 1);
    k_id_compact<<<1, 1, 0, st>>>(T, bin_of, ids, nbins);
    const unsigned NB = get1(c, nbins);
    b.bin_ids.resize(size_t(NB) * 20);
    if (NB) STG_CUDA(cudaMemcpyAsync(b.bin_ids.data(), ids, size_t(NB) * 20, cudaMemcpyDeviceToHost, st));
    b.n_samples = nl;
    b.rank_ids.clear();
    b.rank_sample_off.assign(1, 0);
    b.n_frames = 0;
    if (!nl) {
        STG_CUDA(cudaStreamSynchronize(st));
        return;
    }
    // ranks ascending, file order within a rank: stable radix sort of the line order
    int* key_s = dbuf<int>(c, "bs_key_s", nl);
    uint32_t* ord = dbuf<uint32_t>(c, "bs_ord", nl);
    uint32_t* ord_s = dbuf<uint32_t>(c, "bs_ord_s", nl);
    k_iota_u32<<<grid_of(nl), kT, 0, st>>>(nl, ord);
    size_t tb = 0;
    STG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key_s, ord, ord_s, int64_t(nl), 0, 32, st));
    STG_CUDA(cub::DeviceRadixSort::SortPairs(c.buf("bd_tmp").get(tb), tb, key, key_s, ord, ord_s, int64_t(nl), 0, 32,
                                             st));
    // rank runs
    int* runs = dbuf<int>(c, "bs_runs", nl);
    unsigned long long* rlen = dbuf<unsigned long long>(c, "bs_rlen", nl);
    unsigned long long* nruns = dbuf<unsigned long long>(c, "bs_nruns", 1);
    tb = 0;
    STG_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, key_s, runs, rlen, nruns, int64_t(nl), st));
    STG_CUDA(cub::DeviceRunLengthEncode::Encode(c.buf("bd_tmp").get(tb), tb, key_s, runs, rlen, nruns, int64_t(nl),
                                                st));
    const uint64_t R = get1(c, nruns);
    b.rank_ids.resize(R);
    std::vector<unsigned long long> h_len(R);
    STG_CUDA(cudaMemcpyAsync(b.rank_ids.data(), runs, R * 4, cudaMemcpyDeviceToHost, st));
    STG_CUDA(cudaMemcpyAsync(h_len.data(), rlen, R * 8, cudaMemcpyDeviceToHost, st));
    // frame offsets in sorted order
    uint64_t* nf = dbuf<uint64_t>(c, "bs_nf", nl + 1);
    k_sorted_nf<<<grid_of(nl + 1), kT, 0, st>>>(nl, ord_s, out, nf);
    uint64_t* foff = dbuf<uint64_t>(c, "bd_foff", nl + 1);
    tb = 0;
    STG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, nf, foff, int64_t(nl + 1), st));
    STG_CUDA(cub::DeviceScan::ExclusiveSum(c.buf("bd_tmp").get(tb), tb, nf, foff, int64_t(nl + 1), st));
    const uint64_t F = get1(c, foff + nl);
    for (uint64_t r = 0; r < R; ++r) b.rank_sample_off.push_back(b.rank_sample_off.back() + h_len[r]);
    int64_t* ts = dbuf<int64_t>(c, "bd_ts", nl);
    uint64_t* pc = dbuf<uint64_t>(c, "bd_pc", F + 4);      // 32-byte aligned base (cudaMalloc)
    uint16_t* bn = dbuf<uint16_t>(c, "bd_bin", F + 8);
    k_samples_b<<<grid_of(nl), kT, 0, st>>>(d, nl, ord_s, lines, le, out, foff, T, bin_of, ts, pc, bn);
    STG_CUDA(cudaGetLastError());
    STG_CUDA(cudaStreamSynchronize(st));
    b.n_frames = F;
    b.ts = ts;
    b.foff = foff;
    b.pc = pc;
    b.bin = bn;
}

void bundle_decode_collectives(Ctx& c, const uint8_t* d, uint64_t size, BundleBulk& b) {
    cudaStream_t st = c.stream;
    const uint64_t *ls, *le;
    const uint32_t* lines;
    uint64_t n_all;
    const uint64_t nl = index_lines(c, "bc", d, size, ls, le, lines, n_all);
    int32_t* rank = dbuf<int32_t>(c, "bd_c_rank", nl);
    int32_t* group = dbuf<int32_t>(c, "bd_c_group", nl);
    uint8_t* kind = dbuf<uint8_t>(c, "bd_c_kind", nl);
    int64_t* entry = dbuf<int64_t>(c, "bd_c_entry", nl);
    int64_t* exit_ = dbuf<int64_t>(c, "bd_c_exit", nl);
    int64_t* dur = dbuf<int64_t>(c, "bd_c_dur", nl);
    CollOut* co = dbuf<CollOut>(c, "bc_out", nl);
    unsigned long long* ferr = dbuf<unsigned long long>(c, "bc_err", 1);
    STG_CUDA(cudaMemsetAsync(ferr, 0xff, 8, st));
    if (nl) k_colls<<<grid_of(nl), kT, 0, st>>>(d, nl, lines, ls, le, rank, group, kind, entry, exit_, dur, co, ferr);
    STG_CUDA(cudaGetLastError());
    const unsigned long long e = get1(c, ferr);
    if (e != ~0ull) {
        CollOut o;
        uint32_t L;
        uint64_t s0;
        STG_CUDA(cudaMemcpyAsync(&o, co + e, sizeof o, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaMemcpyAsync(&L, lines + e, 4, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
        STG_CUDA(cudaMemcpyAsync(&s0, ls + L, 8, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
        if (o.err == E_KIND) {
            std::string kind(o.kind_len, '\0');
            if (o.kind_len)
                STG_CUDA(cudaMemcpy(kind.data(), d + s0 + o.kind_s0_rel, o.kind_len, cudaMemcpyDeviceToHost));
            fail(STG_EINVAL, "unknown collective kind: " + kind);
        }
        fail(STG_EINVAL, "collectives.jsonl line " + std::to_string(L + 1) + ": " + what(o.err));
    }
    b.n_coll = nl;
    b.c_rank = rank;
    b.c_group = group;
    b.c_kind = kind;
    b.c_entry = entry;
    b.c_exit = exit_;
    b.c_dur = dur;
}

}  // namespace stg
