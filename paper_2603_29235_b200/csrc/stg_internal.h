// stg_internal.h — shared host/device declarations of libstg.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "stg.h"

namespace stg {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }
#define STG_CUDA(x)                                                                   \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            cudaGetLastError(); /* leave no error state behind for the host app */   \
            ::stg::fail(STG_ECUDA, std::string(#x " -> ") + cudaGetErrorString(e_));  \
        }                                                                             \
    } while (0)

// --------------------------------------------------------- device tables
// One staged symbol table (the device form of a SymbolFile, symfile.hpp:20-41).
// e[i] = {start, size (low 32 bits) | name rank (high 32 bits)}, 16 bytes, so a
// probe and the final entry fetch are single 16-byte loads.  bucket[b] is the
// index of the last entry whose start <= base + (b << shift); the search for an
// offset in bucket b is confined to [bucket[b], bucket[b+1]].
struct DevTable {
    const ulonglong2* e;
    const uint32_t* bucket;
    uint64_t base;
    uint64_t last_start;
    uint32_t shift;
    uint32_t nb;
    uint32_t n;
    uint32_t valid;
};

constexpr uint32_t kUnknownBit = 0x80000000u;
constexpr int kMaxSmemBins = 64;

// Per-rank hash-table slot of the fused symbolize+aggregate kernel.
struct __align__(32) AggSlot {
    unsigned long long hi;  // 0 = empty
    unsigned long long lo;  // fingerprint half 2 (never 0 once written)
    unsigned int count;
    unsigned int rep;       // sample index (rank-relative) that created the slot
    unsigned int pad0, pad1;
};

// Global sequence-dedupe slot.
struct __align__(32) SeqSlot {
    unsigned long long hi;
    unsigned long long lo;
    unsigned int gid;       // 0xffffffff until published
    unsigned int pad;
    unsigned long long rep; // global sample index of the representative
};

// Prefix cache slot: raw non-leaf chain fingerprint -> Σ symbolized terms.
struct __align__(32) PfxSlot {
    unsigned long long hi, lo, ta, tb;
};

// Unknown-frame set slot: (bin, pc) -> slot index.
struct __align__(16) UnkSlot {
    unsigned long long pc;
    unsigned int bin1;      // bin+1; 0 = empty, 0xffffffff = being written
    unsigned int pad;
};

// ------------------------------------------------------------ host-side
// One ingested SYMR table (symtab.cu).  Entries, names and the search index
// live on the device; the host keeps the identity and the search bounds.
struct HostTable {
    uint8_t id[20];
    uint32_t n = 0;
    uint64_t first_start = 0, last_start = 0;
    uint64_t strtab_off = 0;
    uint8_t* d_payload = nullptr;     // the SYMR bytes (name strings are read from here)
    uint32_t* d_name_off = nullptr;   // first name byte of entry i, relative to the string table
    uint32_t* d_name_len = nullptr;
    ulonglong2* d_e = nullptr;        // {start, size | name_rank << 32}
    uint32_t* d_bucket = nullptr;
    uint32_t shift = 0, nb = 0;
    uint64_t dict_version = ~0ull;    // dictionary the ranks in d_e refer to
    HostTable() = default;
    HostTable(const HostTable&) = delete;
    HostTable& operator=(const HostTable&) = delete;
    ~HostTable();
};

// The sorted name dictionary: every loaded table's distinct names in byte-wise
// order (std::string operator<), concatenated; name i = blob[off[i], off[i+1]).
struct Dict {
    std::string blob;
    std::vector<uint64_t> off{0};
    size_t size() const { return off.size() - 1; }
    std::string_view operator[](size_t i) const {
        return std::string_view(blob.data() + off[i], size_t(off[i + 1] - off[i]));
    }
    size_t lower_bound(std::string_view s) const;
};

// Grow-only device buffer.
struct DBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            size_t c = bytes + bytes / 4 + 256;
            if (cudaMalloc(&p, c) != cudaSuccess) {
                cap = 0;
                cudaGetLastError();
                fail(STG_ENOMEM, "device allocation of " + std::to_string(c) + " bytes failed");
            }
            cap = c;
        }
        return p;
    }
    template <class T>
    T* as(size_t n) { return static_cast<T*>(get(n * sizeof(T) + 16)); }
    ~DBuf() {
        if (p) cudaFree(p);
    }
};

struct Result;  // defined in stg_window.cu
struct Bundle;  // bundle.h

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // independent side stages overlapped with k_sym_agg
    std::mutex mu;
    std::vector<std::unique_ptr<HostTable>> tables;
    std::map<std::string, size_t> table_by_id;  // raw 20-byte id -> index
    // sorted name dictionary over all loaded tables (device copy: bufs
    // "dict_blob" / "dict_off", valid for dict_version)
    Dict dict;
    uint64_t dict_version = 0;
    bool dict_dirty = true;
    uint64_t dict_hash = 0, dict_hash_version = ~0ull, dict_agreed_version = ~0ull;
    std::map<std::string, DBuf> bufs;
    DBuf& buf(const std::string& k) { return bufs[k]; }
    std::unique_ptr<Result> result;
    // last loaded bundle (stg_bundle_load); its bulk arrays live in bufs "bd_*"
    std::shared_ptr<Bundle> bundle;
    // bundle file upload threads: pinned double buffers + a stream each
    struct Uploader {
        cudaStream_t stream = nullptr;
        void* pin[2] = {nullptr, nullptr};
        cudaEvent_t ev[2] = {nullptr, nullptr};
    };
    std::vector<Uploader> up;
    // last aggregate_samples result (stg_samples.cu), device-resident
    bool ag_valid = false, ag_exact = false;
    uint64_t ag_windows = 0, ag_records = 0;
    uint64_t ag_cap_hint = 1u << 16;  // table slots the last call needed
    // table-size hints carried from one window to the next (per context, so
    // guarded by mu like everything else here)
    std::vector<uint32_t> hint_rank_used;  // aggregation slots each rank used
    uint32_t hint_pfx_misses = 0;          // prefix-cache misses (distinct raw chains)
    uint32_t hint_unk_used = 0;            // distinct unresolved frames
    uint32_t hint_gid = 0;                 // distinct fingerprints across ranks
    // unknown label -> (position in the dictionary, equals a real name), for dict_version
    std::unordered_map<std::string, std::pair<uint64_t, bool>> label_pos;
    uint64_t label_pos_version = ~0ull;
    // distributed mode (stg_dist_init): one NCCL communicator per context
    void* comm = nullptr;  // ncclComm_t
    int world = 1, wrank = 0;
    ~Ctx();
};

// symtab.cpp
void symtab_ingest(Ctx& c, const uint8_t* claimed_id, const uint8_t* bytes, uint64_t len,
                   int* stored);
void symtab_refresh_dictionary(Ctx& c);  // (re)build dict + stage device tables
std::string hex_id(const uint8_t* id);
std::string unknown_label(const uint8_t* id, uint64_t off);

// device helpers implemented in stg_window.cu
void launch_build_buckets(const ulonglong2* e, uint32_t n, uint64_t base, uint32_t shift,
                          uint32_t nb, uint32_t* bucket, cudaStream_t s);

}  // namespace stg
