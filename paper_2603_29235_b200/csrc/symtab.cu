// symtab.cu — ingest of SYMR symbol tables and the sorted name space, on the GPU
// (SURVEY.md §8(a) a3-a5 and §8(f) row 2).
//
// Replaces parse_symbols (proj/core/src/symfile.cpp:117-157) and the load/ingest
// half of SymbolRepository (symrepo.cpp:35-97).  The 36-byte header is checked
// on the host; the payload is copied to HBM once and
//   k_symr_parse   thread per entry: the reference's per-entry checks in its
//                  order (first failing entry wins, then its first failing
//                  check), {start, size} written straight into the 16-byte
//                  device entries e[i] = {start, size | name_rank << 32}.
// The dictionary (every loaded table's names, byte-wise sorted, unique) is then
// built on the device at the next refresh:
//   k_name_keys    key per entry = (first 8 name bytes big-endian, table:entry)
//   merge sort     NameLess: prefix compare, full byte compare on ties
//   k_name_heads   run heads (a name differs from its predecessor) -> scan = rank
//   k_name_ranks   e[i].y |= rank << 32 for every entry of every table
//   k_dict_gather  the unique names' bytes into one blob (warp per name)
// Ranks order like std::string compares (folded.cpp:18 relies on
// std::map<std::vector<std::string>> order), so folded lines sort on the device
// by rank sequences alone.  The host keeps the blob + offsets (Dict) for name
// rendering; no per-name host work remains.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "stg_internal.h"

namespace stg {

namespace {
constexpr size_t kHeader = 36;
constexpr size_t kEntry = 16;
constexpr int kT = 256;

uint32_t get_u32(const uint8_t* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

inline unsigned grid_of(uint64_t n) {
    uint64_t g = (n + kT - 1) / kT;
    return unsigned(g < 1 ? 1 : (g > 148ull * 64 ? 148ull * 64 : g));
}

// Per-entry checks of parse_symbols in the reference's order; err gets
// min(i * 4 + code) with code 1 = not strictly sorted, 2 = name offset out of
// range, 3 = name out of range.
__global__ void k_symr_parse(const uint8_t* b, uint32_t n, uint64_t strtab_len, ulonglong2* e, uint32_t* name_off,
                             uint32_t* name_len, unsigned long long* err) {
    const uint8_t* strtab = b + kHeader + uint64_t(n) * kEntry;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t* q = reinterpret_cast<const uint32_t*>(b + kHeader + i * kEntry);  // 4-byte aligned
        const uint64_t start = uint64_t(q[0]) | uint64_t(q[1]) << 32;
        const uint32_t sz = q[2], no = q[3];
        unsigned code = 0;
        uint32_t len = 0;
        if (i > 0 && start <= (uint64_t(q[-4]) | uint64_t(q[-3]) << 32)) {
            code = 1;
        } else if (uint64_t(no) + 2 > strtab_len) {
            code = 2;
        } else {
            len = uint32_t(strtab[no]) | uint32_t(strtab[no + 1]) << 8;
            if (len == 0 || uint64_t(no) + 2 + len > strtab_len) code = 3;
        }
        if (code) atomicMin(err, (unsigned long long)(i * 4 + code));
        e[i] = make_ulonglong2(start, sz);
        name_off[i] = no + 2;  // first name byte, relative to the string table
        name_len[i] = len;
    }
}

// One table's names as seen by the dictionary kernels.
struct TabNames {
    const uint8_t* strtab;
    const uint32_t* name_off;
    const uint32_t* name_len;
    ulonglong2* e;
    uint64_t first;  // global index of entry 0
    uint32_t n;
    uint32_t pad;
};

struct NameKey {
    unsigned long long pre;  // first 8 bytes, big-endian, zero padded
    unsigned long long ref;  // table << 32 | entry
};

__device__ __forceinline__ void name_of(const TabNames* t, unsigned long long ref, const uint8_t*& p, uint32_t& len) {
    const TabNames& tt = t[ref >> 32];
    const uint32_t i = uint32_t(ref);
    p = tt.strtab + tt.name_off[i];
    len = tt.name_len[i];
}

// Byte-wise order, shorter prefix first (std::string operator<): compare
// zero-padded bytes, then lengths.
__device__ __forceinline__ int name_cmp(const TabNames* t, unsigned long long ra, unsigned long long rb, uint32_t from) {
    const uint8_t *pa, *pb;
    uint32_t la, lb;
    name_of(t, ra, pa, la);
    name_of(t, rb, pb, lb);
    const uint32_t m = la > lb ? la : lb;
    for (uint32_t k = from; k < m; ++k) {
        const uint32_t ca = k < la ? pa[k] : 0u, cb = k < lb ? pb[k] : 0u;
        if (ca != cb) return ca < cb ? -1 : 1;
    }
    return la < lb ? -1 : (la > lb ? 1 : 0);
}

struct NameLess {
    const TabNames* t;
    __device__ bool operator()(const NameKey& a, const NameKey& b) const {
        if (a.pre != b.pre) return a.pre < b.pre;
        return name_cmp(t, a.ref, b.ref, 8) < 0;
    }
};

__global__ void k_name_keys(const TabNames* t, uint32_t n_tabs, uint64_t total, NameKey* keys) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < total; g += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t lo = 0, hi = n_tabs - 1;  // table of global entry g
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (t[mid].first <= g) lo = mid; else hi = mid - 1;
        }
        const unsigned long long ref = (uint64_t(lo) << 32) | (g - t[lo].first);
        const uint8_t* p;
        uint32_t len;
        name_of(t, ref, p, len);
        unsigned long long pre = 0;
        for (uint32_t k = 0; k < 8; ++k) pre = (pre << 8) | (k < len ? p[k] : 0u);
        keys[g] = NameKey{pre, ref};
    }
}

__global__ void k_name_heads(const TabNames* t, uint64_t total, const NameKey* keys, uint32_t* head) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < total; g += uint64_t(gridDim.x) * blockDim.x)
        head[g] = (g == 0 || keys[g].pre != keys[g - 1].pre || name_cmp(t, keys[g - 1].ref, keys[g].ref, 8) != 0) ? 1u
                                                                                                                   : 0u;
}

// rank = inclusive scan - 1; every entry gets its name's rank, every unique
// name (run head) its length and source.
__global__ void k_name_ranks(const TabNames* t, uint64_t total, const NameKey* keys, const uint32_t* head,
                             const uint32_t* scan, unsigned long long* u_ref, unsigned long long* u_len) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < total; g += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t rank = scan[g] - 1;
        const unsigned long long ref = keys[g].ref;
        const TabNames& tt = t[ref >> 32];
        const uint32_t i = uint32_t(ref);
        tt.e[i].y = (tt.e[i].y & 0xffffffffull) | (uint64_t(rank) << 32);
        if (head[g]) {
            u_ref[rank] = ref;
            u_len[rank] = tt.name_len[i];
        }
    }
}

__global__ void k_dict_gather(const TabNames* t, uint64_t U, const unsigned long long* u_ref,
                              const unsigned long long* off, uint8_t* blob) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t u = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; u < U; u += nw) {
        const uint8_t* p;
        uint32_t len;
        name_of(t, u_ref[u], p, len);
        uint8_t* o = blob + off[u];
        for (uint32_t k = lane; k < len; k += 32) o[k] = p[k];
    }
}

template <class T>
T* dbuf(Ctx& c, const char* name, size_t n) { return c.buf(name).as<T>(n); }

}  // namespace

std::string hex_id(const uint8_t* id) {
    static const char* d = "0123456789abcdef";
    std::string s(40, '0');
    for (int i = 0; i < 20; ++i) {
        s[2 * i] = d[id[i] >> 4];
        s[2 * i + 1] = d[id[i] & 15];
    }
    return s;
}

// unknown_frame_label (symfile.cpp:159-163): "[" + hex id + "+0x" + hex(off) + "]"
std::string unknown_label(const uint8_t* id, uint64_t off) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%llx", (unsigned long long)off);
    return "[" + hex_id(id) + "+0x" + buf + "]";
}

size_t Dict::lower_bound(std::string_view s) const {
    size_t lo = 0, hi = size();
    while (lo < hi) {
        const size_t mid = (lo + hi) / 2;
        if ((*this)[mid] < s) lo = mid + 1; else hi = mid;
    }
    return lo;
}

HostTable::~HostTable() {
    if (d_e) cudaFree(d_e);
    if (d_bucket) cudaFree(d_bucket);
    if (d_payload) cudaFree(d_payload);
    if (d_name_off) cudaFree(d_name_off);
    if (d_name_len) cudaFree(d_name_len);
}

void symtab_ingest(Ctx& c, const uint8_t* claimed_id, const uint8_t* b, uint64_t size, int* stored) {
    // IngestOutcome::AlreadyPresent is decided before any validation
    // (symrepo.cpp:38).
    if (claimed_id) {
        std::string key(reinterpret_cast<const char*>(claimed_id), 20);
        if (c.table_by_id.count(key)) {
            if (stored) *stored = 0;
            return;
        }
    }
    // parse_symbols (symfile.cpp:117-157): header checks, same order and messages
    if (size < kHeader) fail(STG_EINVAL, "symbol file truncated header");
    if (std::memcmp(b, "SYMR", 4) != 0) fail(STG_EINVAL, "symbol file bad magic");
    const uint32_t version = get_u32(b + 4);
    if (version != 1) fail(STG_EINVAL, "unsupported symbol file version " + std::to_string(version));
    const uint32_t n = get_u32(b + 28);
    const uint32_t strtab_off = get_u32(b + 32);
    if (uint64_t(strtab_off) != kHeader + uint64_t(n) * kEntry || strtab_off > size)
        fail(STG_EINVAL, "symbol file bad string-table offset");
    const uint64_t strtab_len = size - strtab_off;

    auto t = std::make_unique<HostTable>();
    std::memcpy(t->id, b + 8, 20);
    t->n = n;
    t->strtab_off = strtab_off;
    cudaStream_t st = c.stream;
    // entries on the device
    STG_CUDA(cudaMalloc(&t->d_payload, size_t(size) + 16));
    STG_CUDA(cudaMemcpyAsync(t->d_payload, b, size, cudaMemcpyHostToDevice, st));
    if (n > 0) {
        STG_CUDA(cudaMalloc(&t->d_e, size_t(n) * sizeof(ulonglong2)));
        STG_CUDA(cudaMalloc(&t->d_name_off, size_t(n) * 4));
        STG_CUDA(cudaMalloc(&t->d_name_len, size_t(n) * 4));
        unsigned long long* err = dbuf<unsigned long long>(c, "sy_err", 1);
        STG_CUDA(cudaMemsetAsync(err, 0xff, 8, st));
        k_symr_parse<<<grid_of(n), kT, 0, st>>>(t->d_payload, n, strtab_len, t->d_e, t->d_name_off, t->d_name_len,
                                                err);
        STG_CUDA(cudaGetLastError());
        unsigned long long e;
        STG_CUDA(cudaMemcpyAsync(&e, err, 8, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
        if (e != ~0ull) {
            const unsigned code = unsigned(e & 3);
            fail(STG_EINVAL, code == 1 ? "symbol entries not strictly sorted"
                             : code == 2 ? "symbol name offset out of range"
                                         : "symbol name out of range");
        }
        // first and last start (the table's search bounds)
        uint64_t fl[2];
        std::memcpy(&fl[0], b + kHeader, 8);
        std::memcpy(&fl[1], b + kHeader + size_t(n - 1) * kEntry, 8);
        t->first_start = fl[0];
        t->last_start = fl[1];
        // bucket index: about four buckets per entry (short in-bucket searches)
        const uint64_t span = t->last_start - t->first_start;
        uint32_t shift = 0;
        while (shift < 63 && (span >> shift) > uint64_t(n) * 4) ++shift;
        t->shift = shift;
        t->nb = uint32_t((span >> shift) + 1);
        STG_CUDA(cudaMalloc(&t->d_bucket, (size_t(t->nb) + 1) * sizeof(uint32_t)));
        launch_build_buckets(t->d_e, n, t->first_start, t->shift, t->nb, t->d_bucket, st);
        STG_CUDA(cudaGetLastError());
    } else {
        STG_CUDA(cudaStreamSynchronize(st));
    }
    std::string key(reinterpret_cast<const char*>(t->id), 20);
    if (claimed_id && std::memcmp(claimed_id, t->id, 20) != 0)
        fail(STG_EINVAL, "symbol file build id does not match ingest key");
    if (c.table_by_id.count(key)) {  // header id already present
        if (stored) *stored = 0;
        return;
    }
    c.table_by_id.emplace(key, c.tables.size());
    c.tables.push_back(std::move(t));
    c.dict_dirty = true;
    if (stored) *stored = 1;
}

// Builds the byte-wise sorted dictionary of every loaded table's names and
// patches each table's entries with ranks into it (all on the device).
void symtab_refresh_dictionary(Ctx& c) {
    if (!c.dict_dirty) return;
    cudaStream_t st = c.stream;
    std::vector<TabNames> tn;
    uint64_t total = 0;
    for (auto& tp : c.tables) {
        HostTable& t = *tp;
        tn.push_back(TabNames{t.d_payload + t.strtab_off, t.d_name_off, t.d_name_len, t.d_e, total, t.n, 0});
        total += t.n;
    }
    Dict& d = c.dict;
    d.blob.clear();
    d.off.assign(1, 0);
    if (total > 0) {
        TabNames* d_tn = dbuf<TabNames>(c, "sy_tabs", tn.size());
        STG_CUDA(cudaMemcpyAsync(d_tn, tn.data(), tn.size() * sizeof(TabNames), cudaMemcpyHostToDevice, st));
        NameKey* keys = dbuf<NameKey>(c, "sy_keys", total);
        k_name_keys<<<grid_of(total), kT, 0, st>>>(d_tn, uint32_t(tn.size()), total, keys);
        size_t tb = 0;
        NameLess less{d_tn};
        STG_CUDA(cub::DeviceMergeSort::SortKeys(nullptr, tb, keys, int64_t(total), less, st));
        STG_CUDA(cub::DeviceMergeSort::SortKeys(c.buf("sy_tmp").get(tb), tb, keys, int64_t(total), less, st));
        uint32_t* head = dbuf<uint32_t>(c, "sy_head", total);
        uint32_t* scan = dbuf<uint32_t>(c, "sy_scan", total);
        k_name_heads<<<grid_of(total), kT, 0, st>>>(d_tn, total, keys, head);
        tb = 0;
        STG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, head, scan, int64_t(total), st));
        STG_CUDA(cub::DeviceScan::InclusiveSum(c.buf("sy_tmp").get(tb), tb, head, scan, int64_t(total), st));
        uint32_t U = 0;
        STG_CUDA(cudaMemcpyAsync(&U, scan + total - 1, 4, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
        if (U >= kUnknownBit) fail(STG_EINVAL, "too many distinct symbol names");
        auto* u_ref = dbuf<unsigned long long>(c, "sy_uref", U);
        auto* u_len = dbuf<unsigned long long>(c, "sy_ulen", U + 1);
        k_name_ranks<<<grid_of(total), kT, 0, st>>>(d_tn, total, keys, head, scan, u_ref, u_len);
        STG_CUDA(cudaMemsetAsync(u_len + U, 0, 8, st));
        auto* off = dbuf<unsigned long long>(c, "dict_off", U + 1);
        tb = 0;
        STG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, u_len, off, int64_t(U) + 1, st));
        STG_CUDA(cub::DeviceScan::ExclusiveSum(c.buf("sy_tmp").get(tb), tb, u_len, off, int64_t(U) + 1, st));
        d.off.resize(size_t(U) + 1);
        STG_CUDA(cudaMemcpyAsync(d.off.data(), off, (size_t(U) + 1) * 8, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
        uint8_t* blob = dbuf<uint8_t>(c, "dict_blob", d.off[U] + 1);
        k_dict_gather<<<grid_of(uint64_t(U) * 32), kT, 0, st>>>(d_tn, U, u_ref, off, blob);
        STG_CUDA(cudaGetLastError());
        d.blob.resize(d.off[U]);
        if (d.off[U]) STG_CUDA(cudaMemcpyAsync(d.blob.data(), blob, d.off[U], cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
    }
    c.dict_version++;
    for (auto& tp : c.tables) tp->dict_version = c.dict_version;
    c.dict_dirty = false;
}

}  // namespace stg
