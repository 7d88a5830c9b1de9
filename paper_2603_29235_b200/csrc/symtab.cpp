// symtab.cpp — ingest/load of SYMR symbol tables and the sorted name space.
//
// Replaces parse_symbols (proj/core/src/symfile.cpp:117-157) and the load/ingest
// half of SymbolRepository (symrepo.cpp:35-97): the SYMR byte format is parsed
// with the reference's validation order and messages, then staged on the GPU as
//   starts[n] u64 | ent[n] = size | name_rank << 32 | bucket[nb+1] u32
// where name_rank is the position of the name in the byte-wise sorted dictionary
// of every loaded table.  Ranks order like std::string compares (folded.cpp:18
// relies on std::map<std::vector<std::string>> order), so folded lines can be
// sorted on the device by rank sequences alone.
#include <algorithm>
#include <cstring>
#include <unordered_map>

#include "stg_internal.h"

namespace stg {

namespace {
constexpr size_t kHeader = 36;
constexpr size_t kEntry = 16;
uint32_t get_u32(const uint8_t* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}
uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
    return v;
}
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

void symtab_ingest(Ctx& c, const uint8_t* claimed_id, const uint8_t* b, uint64_t size,
                   int* stored) {
    // IngestOutcome::AlreadyPresent is decided before any validation
    // (symrepo.cpp:38).
    if (claimed_id) {
        std::string key(reinterpret_cast<const char*>(claimed_id), 20);
        if (c.table_by_id.count(key)) {
            if (stored) *stored = 0;
            return;
        }
    }
    // parse_symbols (symfile.cpp:117-157), same checks in the same order.
    if (size < kHeader) fail(STG_EINVAL, "symbol file truncated header");
    if (std::memcmp(b, "SYMR", 4) != 0) fail(STG_EINVAL, "symbol file bad magic");
    uint32_t version = get_u32(b + 4);
    if (version != 1) fail(STG_EINVAL, "unsupported symbol file version " + std::to_string(version));
    uint32_t n = get_u32(b + 28);
    uint32_t strtab_off = get_u32(b + 32);
    if (uint64_t(strtab_off) != kHeader + uint64_t(n) * kEntry || strtab_off > size)
        fail(STG_EINVAL, "symbol file bad string-table offset");
    const uint8_t* strtab = b + strtab_off;
    uint64_t strtab_len = size - strtab_off;

    auto t = std::make_unique<HostTable>();
    std::memcpy(t->id, b + 8, 20);
    t->starts.resize(n);
    t->sizes.resize(n);
    t->name_local.resize(n);
    std::unordered_map<std::string, uint32_t> local;
    uint64_t prev = 0;
    for (uint32_t i = 0; i < n; ++i) {
        const uint8_t* p = b + kHeader + size_t(i) * kEntry;
        uint64_t start = get_u64(p);
        uint32_t sz = get_u32(p + 8);
        uint32_t name_off = get_u32(p + 12);
        if (i > 0 && start <= prev) fail(STG_EINVAL, "symbol entries not strictly sorted");
        prev = start;
        if (uint64_t(name_off) + 2 > strtab_len) fail(STG_EINVAL, "symbol name offset out of range");
        uint16_t len = uint16_t(strtab[name_off] | strtab[name_off + 1] << 8);
        if (len == 0 || uint64_t(name_off) + 2 + len > strtab_len)
            fail(STG_EINVAL, "symbol name out of range");
        std::string name(reinterpret_cast<const char*>(strtab + name_off + 2), len);
        auto it = local.find(name);
        uint32_t id;
        if (it == local.end()) {
            id = uint32_t(t->names.size());
            local.emplace(name, id);
            t->names.push_back(std::move(name));
        } else {
            id = it->second;
        }
        t->starts[i] = start;
        t->sizes[i] = sz;
        t->name_local[i] = id;
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
// (re)stages each table on the device with ranks into it.
void symtab_refresh_dictionary(Ctx& c) {
    if (!c.dict_dirty) return;
    std::vector<std::string> all;
    size_t total = 0;
    for (auto& t : c.tables) total += t->names.size();
    all.reserve(total);
    for (auto& t : c.tables)
        for (auto& s : t->names) all.push_back(s);
    // std::string operator< is byte-wise (char_traits<char>::lt compares as
    // unsigned char), shorter prefix first — exactly memcmp + length.
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    if (all.size() >= kUnknownBit) fail(STG_EINVAL, "too many distinct symbol names");
    c.dict = std::move(all);
    c.dict_version++;
    for (auto& tp : c.tables) {
        HostTable& t = *tp;
        std::vector<uint32_t> rank_of(t.names.size());
        for (size_t i = 0; i < t.names.size(); ++i)
            rank_of[i] = uint32_t(std::lower_bound(c.dict.begin(), c.dict.end(), t.names[i]) - c.dict.begin());
        uint32_t n = uint32_t(t.starts.size());
        std::vector<ulonglong2> ent(n);
        for (uint32_t i = 0; i < n; ++i) {
            ent[i].x = t.starts[i];
            ent[i].y = uint64_t(t.sizes[i]) | uint64_t(rank_of[t.name_local[i]]) << 32;
        }
        if (!t.d_e && n > 0) {
            STG_CUDA(cudaMalloc(&t.d_e, n * sizeof(ulonglong2)));
            // bucket index: about four buckets per entry (short in-bucket searches)
            uint64_t span = t.starts[n - 1] - t.starts[0];
            uint32_t shift = 0;
            while (shift < 63 && (span >> shift) > uint64_t(n) * 4) ++shift;
            t.shift = shift;
            t.nb = uint32_t((span >> shift) + 1);
            STG_CUDA(cudaMalloc(&t.d_bucket, (size_t(t.nb) + 1) * sizeof(uint32_t)));
        }
        if (n > 0) {
            STG_CUDA(cudaMemcpyAsync(t.d_e, ent.data(), n * sizeof(ulonglong2), cudaMemcpyHostToDevice, c.stream));
            launch_build_buckets(t.d_e, n, t.starts[0], t.shift, t.nb, t.d_bucket, c.stream);
        }
        t.dict_version = c.dict_version;
        STG_CUDA(cudaStreamSynchronize(c.stream));
    }
    c.dict_dirty = false;
}

}  // namespace stg
