// bench_gen.cu — BENCH INFRASTRUCTURE (libstg_bench.so, not part of libstg):
// deterministic on-device generator of the C2 workload:
// R ranks x N samples, 64-frame stacks over three binaries (python 20 % of
// frames at the root, libtorch 60 %, cuda 20 % at the leaf), a pool of P
// distinct symbolized stacks per rank drawn Zipf(1.1), per-rank rotated
// popularity, call-site offsets fixed per (stack node), leaf offsets uniform
// inside the leaf function (many raw PCs -> one name), and a straggler rank
// whose samples carry a 9-frame softirq path at the leaf with a given share.
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace {

__device__ __forceinline__ uint64_t h64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

struct GenParams {
    uint64_t seed;
    int ranks;
    uint64_t spr;          // samples per rank
    int depth;             // 64
    uint32_t pool;         // distinct stacks per rank
    const double* zipf_cdf;  // [pool]
    const uint64_t* starts[3];
    const uint32_t* sizes[3];
    uint32_t nsym[3];
    uint32_t hot[3];       // functions actually executed per binary
    uint64_t soft_pc[9];   // softirq path (bin 2), root-first
    int slow_rank;
    double soft_share;
    uint32_t jit_per_million;  // samples whose leaf is an unknown JIT frame
    int64_t period_ns;
    const int64_t* skew;   // [ranks]
    int64_t* ts;
    uint64_t* foff;
    uint64_t* pc;
    uint16_t* bin;
};

__device__ __forceinline__ int bin_of_level(int j, int depth) {
    // root-first level j: first 20 % python, next 60 % libtorch, last 20 % cuda
    int a = depth / 5, b = depth - depth / 5;
    return j < a ? 0 : (j < b ? 1 : 2);
}

// Node id of level j of stack p: the first 16 levels branch on the bits of p
// (a binary call tree shared by all stacks), deeper levels continue uniquely.
__device__ __forceinline__ uint64_t node_of(uint64_t seed, uint32_t p, int j) {
    uint32_t bits = j < 16 ? (p & ((1u << j) - 1)) : p;
    return h64(seed ^ (uint64_t(j) << 40) ^ (uint64_t(bits) << 1) ^ (j < 16 ? 0 : 1));
}

__global__ void k_gen(GenParams g) {
    const uint64_t n = uint64_t(g.ranks) * g.spr;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const int r = int(i / g.spr);
        const uint64_t k = i % g.spr;
        uint64_t u = h64(g.seed ^ (i * 0x2545f4914f6cdd1dull));
        // Zipf draw by inverse CDF
        double x = double(u >> 11) * (1.0 / 9007199254740992.0);
        uint32_t lo = 0, hi = g.pool - 1;
        while (lo < hi) {
            uint32_t m = (lo + hi) >> 1;
            if (g.zipf_cdf[m] < x) lo = m + 1; else hi = m;
        }
        uint32_t p = (lo + uint32_t(r) * 7919u) % g.pool;  // per-rank rotated popularity
        bool soft = r == g.slow_rank && double(h64(u) >> 11) * (1.0 / 9007199254740992.0) < g.soft_share;
        bool jit = !soft && (h64(u ^ 0x77) % 1000000ull) < g.jit_per_million;
        const int D = g.depth;
        g.ts[i] = int64_t(k) * g.period_ns + int64_t(h64(u ^ 0x55) % uint64_t(g.period_ns / 50 + 1)) + g.skew[r];
        g.foff[i] = i * uint64_t(D);
        if (i == n - 1) g.foff[n] = n * uint64_t(D);
        uint64_t* out_pc = g.pc + i * uint64_t(D);
        uint16_t* out_bin = g.bin + i * uint64_t(D);
        // leaf first: position q = D-1-j for root-first level j
        for (int j = 0; j < D; ++j) {
            int q = D - 1 - j;
            uint64_t pcv;
            uint16_t b;
            if (soft && j >= D - 9) {
                b = 2;
                pcv = g.soft_pc[j - (D - 9)];
            } else if (jit && j == D - 1) {
                b = 3;  // binary without a symbol file
                pcv = 0x7f0000000000ull + (h64(u ^ 0x99) % 1000) * 16;
            } else {
                b = uint16_t(bin_of_level(j, D));
                uint64_t node = node_of(g.seed, p, j);
                uint32_t f = uint32_t(node % g.hot[b]);
                f = uint32_t((uint64_t(f) * 2654435761ull) % g.nsym[b]);  // spread hot set over the table
                uint64_t st = g.starts[b][f];
                uint32_t sz = g.sizes[b][f];
                uint64_t off = (j == D - 1 || (soft && j == D - 10)) ? h64(u ^ uint64_t(j)) % sz
                                                                     : h64(node ^ 0x1234) % sz;
                pcv = st + off;
            }
            out_pc[q] = pcv;
            out_bin[q] = b;
        }
    }
}

}  // namespace

extern "C" int bench_gen_c2(uint64_t seed, int ranks, uint64_t spr, int depth, uint32_t pool,
                            const double* zipf_cdf, const uint64_t* const* starts,
                            const uint32_t* const* sizes, const uint32_t* nsym, const uint32_t* hot,
                            const uint64_t* soft_pc, int slow_rank, double soft_share,
                            uint32_t jit_per_million, int64_t period_ns, const int64_t* skew, int64_t* ts,
                            uint64_t* foff, uint64_t* pc, uint16_t* bin, void* stream) {
    GenParams g{};
    g.seed = seed;
    g.ranks = ranks;
    g.spr = spr;
    g.depth = depth;
    g.pool = pool;
    g.zipf_cdf = zipf_cdf;
    for (int b = 0; b < 3; ++b) {
        g.starts[b] = starts[b];
        g.sizes[b] = sizes[b];
        g.nsym[b] = nsym[b];
        g.hot[b] = hot[b];
    }
    for (int j = 0; j < 9; ++j) g.soft_pc[j] = soft_pc[j];
    g.slow_rank = slow_rank;
    g.soft_share = soft_share;
    g.jit_per_million = jit_per_million;
    g.period_ns = period_ns;
    g.skew = skew;
    g.ts = ts;
    g.foff = foff;
    g.pc = pc;
    g.bin = bin;
    k_gen<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(g);
    return int(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Bundle writer for `bench.py --config bundle`: samples.jsonl and
// collectives.jsonl exactly as write_bundle emits them (nlohmann dump of
// sample_to_json / the collective record, keys in sorted order, bundle.cpp:31-42,
// 128-139) from host SoA arrays.
#include <cstdio>
#include <string>
#include <vector>

extern "C" int bench_write_jsonl(const char* samples_path, const char* coll_path, int n_ranks, const int32_t* rank_ids,
                                 const uint64_t* rank_off, const int64_t* ts, const uint64_t* foff, const uint64_t* pc,
                                 const uint16_t* bin, int n_bins, const uint8_t* bin_ids, uint64_t n_coll,
                                 const int32_t* c_rank, const int32_t* c_group, const uint8_t* c_kind,
                                 const int64_t* c_entry, const int64_t* c_exit, const int64_t* c_dur) {
    static const char* kinds[] = {"AllReduce", "ReduceScatter", "AllGather", "Broadcast", "P2P"};
    static const char* hexd = "0123456789abcdef";
    std::vector<std::string> hx(static_cast<size_t>(n_bins));
    for (int b = 0; b < n_bins; ++b)
        for (int j = 0; j < 20; ++j) {
            hx[size_t(b)] += hexd[bin_ids[20 * b + j] >> 4];
            hx[size_t(b)] += hexd[bin_ids[20 * b + j] & 15];
        }
    FILE* f = std::fopen(samples_path, "wb");
    if (!f) return 1;
    std::string line;
    char num[32];
    for (int r = 0; r < n_ranks; ++r)
        for (uint64_t s = rank_off[r]; s < rank_off[r + 1]; ++s) {
            line.assign("{\"frames\":[");
            for (uint64_t k = foff[s]; k < foff[s + 1]; ++k) {
                if (k > foff[s]) line += ',';
                line += "[\"";
                line += hx[bin[k]];
                line += "\",";
                std::snprintf(num, sizeof num, "%llu", (unsigned long long)pc[k]);
                line += num;
                line += ']';
            }
            std::snprintf(num, sizeof num, "%d", rank_ids[r]);
            line += "],\"rank\":";
            line += num;
            line += ",\"spaces\":\"";
            line.append(size_t(foff[s + 1] - foff[s]), 'u');
            std::snprintf(num, sizeof num, "%d", 1000 + rank_ids[r]);
            line += "\",\"thread\":";
            line += num;
            std::snprintf(num, sizeof num, "%lld", (long long)ts[s]);
            line += ",\"ts\":";
            line += num;
            line += "}\n";
            std::fwrite(line.data(), 1, line.size(), f);
        }
    std::fclose(f);
    f = std::fopen(coll_path, "wb");
    if (!f) return 1;
    for (uint64_t i = 0; i < n_coll; ++i)
        std::fprintf(f, "{\"entry\":%lld,\"exit\":%lld,\"gpu_duration\":%lld,\"group\":%d,\"kind\":\"%s\",\"rank\":%d}\n",
                     (long long)c_entry[i], (long long)c_exit[i], (long long)c_dur[i], c_group[i], kinds[c_kind[i]],
                     c_rank[i]);
    std::fclose(f);
    return 0;
}
