// stg_window.cu — the per-window batch on the GPU: replaces build_group_data
// (proj/core/src/bundle.cpp:252-324) and the statistics behind diagnose
// (diagnosis.cpp:76-111, 122-263).  Stage map:
//   d  collectives: k_coll_* (match_collectives collective.cpp:29-103,
//      align_clocks :105-125, entry_lateness :127-142, windowing bundle.cpp:270-285)
//      + k_straggler_* (detect_straggler diagnosis.cpp:76-111, bit-exact FP order)
//   a+b samples:   k_sym_agg — fused symbolize (SymbolFile::lookup symfile.cpp:54-75)
//      + aggregate (aggregate_samples samples.cpp:31-85 / to_folded folded.cpp:56-71)
//      keyed by the symbolized stack; k_seq_* dedupe, materialize, sort -> folded
//      lines in std::map order (folded.cpp:11-19)
//   c  diff:        k_incl (inclusive_fractions folded.cpp:45-54), k_waterline
//      (compute_waterline diagnosis.cpp:35-55), candidate kernels for cpu_diff /
//      temporal_diff; the decision ladder of diagnose (diagnosis.cpp:301-432) runs
//      on the host over these device-side summaries.
#include <cub/cub.cuh>
#include <functional>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <sstream>

#include "kernels.cuh"
#include "result.h"

namespace stg {

Ctx::~Ctx() {
    tables.clear();  // HostTable frees its device arrays
    bufs.clear();
    for (auto& u : up) {
        for (int k = 0; k < 2; ++k) {
            if (u.pin[k]) cudaFreeHost(u.pin[k]);
            if (u.ev[k]) cudaEventDestroy(u.ev[k]);
        }
        if (u.stream) cudaStreamDestroy(u.stream);
    }
    if (side) cudaStreamDestroy(side);
    if (stream) cudaStreamDestroy(stream);
}

std::string Result::name_of(uint32_t f) const {
    // unknown labels carry explicit final ranks; real names fill the rest in order
    auto it = std::lower_bound(unk_final.begin(), unk_final.end(), uint64_t(f));
    if (it != unk_final.end() && *it == f) return unk_labels[size_t(it - unk_final.begin())];
    uint64_t before = uint64_t(it - unk_final.begin());
    return std::string((*dict)[f - before]);
}

namespace {

constexpr int kThreads = 256;
inline unsigned grid_for(uint64_t n, int threads = kThreads, unsigned cap = 148 * 32) {
    uint64_t g = (n + threads - 1) / threads;
    if (g == 0) g = 1;
    return unsigned(std::min<uint64_t>(g, cap));
}
inline uint64_t next_pow2(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

// ============================================================== tables
__global__ void k_build_buckets(const ulonglong2* e, uint32_t n, uint64_t base, uint32_t shift,
                                uint32_t nb, uint32_t* bucket) {
    for (uint64_t b = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; b <= nb;
         b += uint64_t(gridDim.x) * blockDim.x) {
        if (b == nb) {
            bucket[b] = n - 1;
            continue;
        }
        uint64_t key = base + (b << shift);
        // last index with starts[i] <= key
        uint32_t lo = 0, hi = n;  // upper_bound
        while (lo < hi) {
            uint32_t mid = (lo + hi) >> 1;
            if (e[mid].x <= key)
                lo = mid + 1;
            else
                hi = mid;
        }
        bucket[b] = lo == 0 ? 0 : lo - 1;
    }
}

// ========================================================= collectives
// Group/kind ranges, so the stream key uses only the bits it needs.
__global__ void k_coll_ranges(uint64_t n, const int32_t* group, const uint8_t* kind, int* gmin, int* gmax, int* kmax) {
    int lo = INT_MAX, hi = INT_MIN, km = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        lo = min(lo, group[i]);
        hi = max(hi, group[i]);
        km = max(km, int(kind[i]));
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        km = max(km, __shfl_xor_sync(0xffffffffu, km, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(gmin, lo);
        atomicMax(gmax, hi);
        atomicMax(kmax, km);
    }
}

// key = (group - gmin) << (kbits + rbits) | kind << rbits | rank: a stable sort
// on it splits events into (group, kind) streams and per-rank runs while keeping
// each rank's input order (collective.cpp:33-43).
// err_rank: set when an event's rank lies outside [rlo, rhi) (a sharded
// context's own ranks; [0, 2^24) otherwise).
__global__ void k_coll_keys(uint64_t n, const int32_t* rank, const int32_t* group, const uint8_t* kind, int gmin,
                            int kbits, int rbits, int rlo, int rhi, uint64_t* key, uint32_t* idx, int* err_rank) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        int32_t r = rank[i];
        if (r < rlo || r >= rhi || r >= (1 << 24)) *err_rank = 1;
        key[i] = (uint64_t(uint32_t(group[i] - gmin)) << (kbits + rbits)) | (uint64_t(kind[i]) << rbits) |
                 uint64_t(uint32_t(r) & 0xffffffu);
        idx[i] = uint32_t(i);
    }
}

__global__ void k_coll_gather(uint64_t n, const uint64_t* key, const uint32_t* idx, const int64_t* entry,
                              const int64_t* exit_, int rbits, int64_t* s_entry, int64_t* s_exit,
                              unsigned long long* err_ee, unsigned long long* err_ord,
                              uint32_t* seg_flag, uint32_t* stream_flag) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
         p += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t e = idx[p];
        int64_t en = entry[e], ex = exit_[e];
        s_entry[p] = en;
        s_exit[p] = ex;
        if (en >= ex) atomicMin(err_ee, (unsigned long long)e);
        bool new_seg = p == 0 || key[p] != key[p - 1];
        bool new_stream = p == 0 || (key[p] >> rbits) != (key[p - 1] >> rbits);
        if (!new_seg && en < entry[idx[p - 1]]) atomicMin(err_ord, (unsigned long long)e);
        seg_flag[p] = new_seg;
        stream_flag[p] = new_stream;
    }
}

// Stream and segment tables on the device (no host round trip): st_seg[s] =
// index of the first segment of stream s (seg_pos is sorted, st_pos a subset of
// it), seg_stream[j] = stream containing segment j.
__global__ void k_stream_tables(const unsigned long long* counts, const uint32_t* seg_pos, const uint32_t* st_pos,
                                uint32_t* st_seg, uint32_t* seg_stream) {
    const uint64_t n_seg = counts[0], n_st = counts[1];
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < n_seg + n_st + 1;
         t += uint64_t(gridDim.x) * blockDim.x) {
        if (t < n_st) {
            const uint32_t v = st_pos[t];
            uint64_t lo = 0, hi = n_seg;
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (seg_pos[mid] < v) lo = mid + 1; else hi = mid;
            }
            st_seg[t] = uint32_t(lo);
        } else if (t == n_st) {
            st_seg[n_st] = uint32_t(n_seg);
        } else {
            const uint64_t j = t - n_st - 1;
            const uint32_t v = seg_pos[j];
            uint64_t lo = 0, hi = n_st;  // upper_bound(st_pos, v) - 1
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (st_pos[mid] <= v) lo = mid + 1; else hi = mid;
            }
            seg_stream[j] = uint32_t(lo - 1);
        }
    }
}
// per-rank segment lists from the segments sorted by rank: rso[r] = first
// position of rank r in the sorted rank list
__global__ void k_rank_offsets(int span, const uint32_t* ranks_sorted, uint64_t n_seg, uint32_t* rso) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= span; r += gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = n_seg;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (ranks_sorted[mid] < uint32_t(r)) lo = mid + 1; else hi = mid;
        }
        rso[r] = uint32_t(lo);
    }
}

// One block per stream: coarse offsets (collective.cpp:49-54), counts.
__global__ void k_coll_streams(int n_streams, const uint32_t* st_seg, const uint32_t* seg_pos,
                               const int64_t* s_entry, int64_t* coarse, uint32_t* kmin, uint32_t* kmax) {
    int s = blockIdx.x;
    if (s >= n_streams) return;
    uint32_t a = st_seg[s], b = st_seg[s + 1];
    __shared__ long long s_min;
    __shared__ unsigned s_kmin, s_kmax;
    if (threadIdx.x == 0) {
        s_min = LLONG_MAX;
        s_kmin = 0xffffffffu;
        s_kmax = 0;
    }
    __syncthreads();
    for (uint32_t j = a + threadIdx.x; j < b; j += blockDim.x) {
        atomicMin(&s_min, (long long)s_entry[seg_pos[j]]);
        uint32_t len = seg_pos[j + 1] - seg_pos[j];
        atomicMin(&s_kmin, len);
        atomicMax(&s_kmax, len);
    }
    __syncthreads();
    for (uint32_t j = a + threadIdx.x; j < b; j += blockDim.x) coarse[j] = s_entry[seg_pos[j]] - s_min;
    if (threadIdx.x == 0) {
        kmin[s] = s_kmin;
        kmax[s] = s_kmax;
    }
}

// Regular-case proof: instance k of a stream is {every rank's k-th event} iff the
// greedy sweep (collective.cpp:64-89) starting from all heads at k pulls them all.
// One warp per (stream, k): seed = min pre-aligned entry, ties to the lowest
// rank (strict <, rank order); then every head must overlap the seed interval.
__global__ void k_coll_regular(int n_streams, const uint32_t* st_seg, const uint32_t* seg_pos,
                               const int64_t* coarse, const int64_t* s_entry, const int64_t* s_exit,
                               const uint32_t* kmin, const uint64_t* k_base, uint64_t n_k,
                               int64_t skew, uint32_t* first_fail) {
    // one warp per (stream, k): lanes stride over the stream's rank segments
    const int lane = threadIdx.x & 31;
    for (uint64_t t = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; t < n_k;
         t += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        int lo = 0, hi = n_streams - 1;  // stream of t: last s with k_base[s] <= t
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (k_base[mid] <= t) lo = mid; else hi = mid - 1;
        }
        const int s = lo;
        const uint32_t k = uint32_t(t - k_base[s]);
        const uint32_t a = st_seg[s], b = st_seg[s + 1];
        // seed: min pre-aligned entry, ties to the lowest segment (rank order)
        long long best = LLONG_MAX;
        uint32_t bj = 0xffffffffu;
        for (uint32_t j = a + lane; j < b; j += 32) {
            const long long e = s_entry[seg_pos[j] + k] - coarse[j];
            if (e < best) {  // j ascends per lane: strict < keeps the lowest
                best = e;
                bj = j;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long ob = __shfl_xor_sync(0xffffffffu, best, o);
            const uint32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (ob < best || (ob == best && oj < bj)) {
                best = ob;
                bj = oj;
            }
        }
        const long long best_exit = s_exit[seg_pos[bj] + k] - coarse[bj];
        bool ok = true;
        for (uint32_t j = a + lane; j < b && ok; j += 32) {
            const uint64_t p = seg_pos[j] + k;
            const long long e = s_entry[p] - coarse[j], x = s_exit[p] - coarse[j];
            ok = e <= best_exit + skew && x + skew >= best;
        }
        ok = __all_sync(0xffffffffu, ok);
        if (!ok && lane == 0) atomicMin(first_fail + s, k);
    }
}

// Regular part: event (j, k<k0) -> local instance k.
__global__ void k_coll_assign_regular(int n_streams, const uint32_t* st_seg, const uint32_t* seg_pos,
                                      const uint32_t* seg_stream, uint32_t n_seg, const uint32_t* k0,
                                      uint32_t* inst_local) {
    for (uint32_t j = blockIdx.x; j < n_seg; j += gridDim.x) {
        uint32_t s = seg_stream[j];
        uint32_t lim = k0[s];
        uint32_t len = seg_pos[j + 1] - seg_pos[j];
        for (uint32_t k = threadIdx.x; k < len; k += blockDim.x)
            inst_local[seg_pos[j] + k] = k < lim ? k : 0xffffffffu;
    }
}

// Sequential greedy sweep for the irregular tail of one stream (one block per
// stream), from heads at k0 — a direct transcription of collective.cpp:64-89.
__global__ void k_coll_sequential(const int* streams, const uint32_t* st_seg, const uint32_t* seg_pos,
                                  const int64_t* coarse, const int64_t* s_entry, const int64_t* s_exit,
                                  const uint32_t* k0, int64_t skew, uint32_t* head_buf,
                                  uint32_t* inst_local, uint32_t* n_inst) {
    int s = streams[blockIdx.x];
    uint32_t a = st_seg[s], b = st_seg[s + 1];
    uint32_t* head = head_buf + a;
    for (uint32_t j = a + threadIdx.x; j < b; j += blockDim.x) head[j - a] = seg_pos[j] + k0[s];
    __shared__ long long r_e[1024];
    __shared__ unsigned r_j[1024];
    __shared__ long long sd_entry, sd_exit;
    __shared__ int done;
    __syncthreads();
    uint32_t inst = k0[s];
    while (true) {
        long long be = LLONG_MAX;
        unsigned bj = 0xffffffffu;
        for (uint32_t j = a + threadIdx.x; j < b; j += blockDim.x) {
            uint32_t h = head[j - a];
            if (h < seg_pos[j + 1]) {
                long long e = s_entry[h] - coarse[j];
                if (e < be || (e == be && j < bj)) {
                    be = e;
                    bj = j;
                }
            }
        }
        r_e[threadIdx.x] = be;
        r_j[threadIdx.x] = bj;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if (threadIdx.x < w) {
                long long oe = r_e[threadIdx.x + w];
                unsigned oj = r_j[threadIdx.x + w];
                if (oe < r_e[threadIdx.x] || (oe == r_e[threadIdx.x] && oj < r_j[threadIdx.x])) {
                    r_e[threadIdx.x] = oe;
                    r_j[threadIdx.x] = oj;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            done = r_j[0] == 0xffffffffu;
            if (!done) {
                uint32_t h = head[r_j[0] - a];
                sd_entry = s_entry[h] - coarse[r_j[0]];
                sd_exit = s_exit[h] - coarse[r_j[0]];
            }
        }
        __syncthreads();
        if (done) break;
        long long se = sd_entry, sx = sd_exit;
        for (uint32_t j = a + threadIdx.x; j < b; j += blockDim.x) {
            uint32_t h = head[j - a];
            if (h < seg_pos[j + 1]) {
                long long e = s_entry[h] - coarse[j], x = s_exit[h] - coarse[j];
                if (e <= sx + skew && x + skew >= se) {
                    inst_local[h] = inst;
                    head[j - a] = h + 1;
                }
            }
        }
        ++inst;
        __syncthreads();
    }
    if (threadIdx.x == 0) n_inst[s] = inst;
}

// Per event: global instance id, instance aggregates.
__global__ void k_coll_inst(uint64_t n, const uint64_t* key, const uint32_t* seg_stream_of_pos_unused,
                            const uint32_t* stream_of_pos, const uint64_t* inst_base,
                            const uint32_t* inst_local, const int64_t* s_exit, const uint8_t* group_member,
                            uint32_t* inst_of, unsigned long long* inst_max_exit, unsigned* inst_size,
                            unsigned* inst_ingroup, uint64_t rmask) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
         p += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t s = stream_of_pos[p];
        uint32_t g = uint32_t(inst_base[s] + inst_local[p]);
        inst_of[p] = g;
        uint32_t r = uint32_t(key[p] & rmask);
        atomicMax((long long*)&inst_max_exit[g], (long long)s_exit[p]);
        atomicAdd(&inst_size[g], 1u);
        if (group_member[r]) atomicAdd(&inst_ingroup[g], 1u);
    }
}

// align_clocks (collective.cpp:105-125) inputs: delta = exit - max exit for
// events of complete instances (flag = 1), min delta for the key width.
// dval = exit - max exit (<= 0) for events of complete instances, +1 for the
// others (the median select skips positive values); min delta for the key width.
__global__ void k_coll_deltas(uint64_t n, const uint32_t* inst_of, const int64_t* s_exit,
                              const unsigned long long* inst_max_exit, const unsigned* inst_ingroup, unsigned n_group,
                              int64_t* dval, long long* dmin) {
    long long lo = 0;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t g = inst_of[p];
        const bool ok = inst_ingroup[g] >= n_group;
        const int64_t d = ok ? s_exit[p] - (long long)inst_max_exit[g] : 1;
        dval[p] = d;
        if (ok) lo = min(lo, (long long)d);
    }
    for (int o = 16; o > 0; o >>= 1) lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    if ((threadIdx.x & 31) == 0) atomicMin(dmin, lo);
}
// align_clocks (collective.cpp:105-125) without sorting the deltas: one CTA per
// rank walks the rank's (stream, rank) segments and finds the two middle order
// statistics of its barrier-exit deltas by radix select (8-bit digits from the
// top, shared-memory histograms, warp-aggregated increments), then takes the
// median exactly like the reference (even count: truncating int64 mean, :122).
__global__ void k_seg_rank(uint64_t n_seg, const uint32_t* seg_pos, const uint64_t* key, uint64_t rmask,
                           uint32_t* seg_rank) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < n_seg; j += uint64_t(gridDim.x) * blockDim.x)
        seg_rank[j] = uint32_t(key[seg_pos[j]] & rmask);
}
constexpr int kMedThreads = 1024;
constexpr int kMedBits = 11, kMedBins = 1 << kMedBits;  // 2 x 8 KB histograms, 2 bins per thread
// block-wide exclusive scan of two counters per thread (1,024 threads)
__device__ __forceinline__ void med_scan2(unsigned a, unsigned b, unsigned& ea, unsigned& eb, unsigned (*ws)[32]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned ta = __shfl_up_sync(0xffffffffu, ia, o), tb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
            ia += ta;
            ib += tb;
        }
    }
    if (lane == 31) {
        ws[0][wid] = ia;
        ws[1][wid] = ib;
    }
    __syncthreads();
    if (wid == 0) {
        unsigned xa = ws[0][lane], xb = ws[1][lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned ta = __shfl_up_sync(0xffffffffu, xa, o), tb = __shfl_up_sync(0xffffffffu, xb, o);
            if (lane >= o) {
                xa += ta;
                xb += tb;
            }
        }
        ws[0][lane] = xa;
        ws[1][lane] = xb;
    }
    __syncthreads();
    ea = ia - a + (wid ? ws[0][wid - 1] : 0u);
    eb = ib - b + (wid ? ws[1][wid - 1] : 0u);
}
__global__ void __launch_bounds__(kMedThreads) k_coll_median_sel(int rank_span, const uint32_t* rso, const uint32_t* rsegs,
                                                                 const uint32_t* seg_pos, const int64_t* dval,
                                                                 const long long* dmin_p, int64_t* off,
                                                                 uint8_t* has_off, unsigned long long* n_total) {
    __shared__ unsigned hist[2][kMedBins];
    __shared__ unsigned s_ws[2][32];
    __shared__ unsigned long long s_pref[2], s_k[2], s_cnt;
    const int lane = threadIdx.x & 31;
    constexpr int U = 4;  // elements per thread per step: U loads in flight
    const long long dmin = *dmin_p;  // min delta (<= 0): the keys are v - dmin in [0, -dmin]
    const int dbits = dmin < 0 ? 64 - __clzll((unsigned long long)(-dmin)) : 1;
    const int nd = (dbits + kMedBits - 1) / kMedBits;
    for (int r = blockIdx.x; r < rank_span; r += gridDim.x) {
        const uint32_t j0 = rso[r], j1 = rso[r + 1];
        if (threadIdx.x == 0) {
            s_pref[0] = s_pref[1] = 0;
            s_cnt = 0;
        }
        bool first = true;
        for (int sh = (nd - 1) * kMedBits; sh >= 0; sh -= kMedBits) {
            for (int t = threadIdx.x; t < 2 * kMedBins; t += blockDim.x) (&hist[0][0])[t] = 0;
            __syncthreads();
            const unsigned long long p0 = (s_pref[0] >> sh) >> kMedBits, p1 = (s_pref[1] >> sh) >> kMedBits;
            unsigned long long c = 0;
            for (uint32_t j = j0; j < j1; ++j) {
                const uint32_t a = seg_pos[rsegs[j]], b = seg_pos[rsegs[j] + 1];
                for (uint32_t q0 = a; q0 < b; q0 += U * kMedThreads) {  // warp-uniform trip count
                    int64_t v[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const uint32_t q = q0 + u * kMedThreads + threadIdx.x;
                        v[u] = q < b ? dval[q] : 1;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        unsigned d0 = 0xffffffffu, d1 = 0xffffffffu;
                        if (v[u] <= 0) {  // a delta of a complete instance
                            ++c;
                            const unsigned long long x = (unsigned long long)(v[u] - dmin) >> sh;
                            const unsigned dg = unsigned(x) & (kMedBins - 1);
                            if ((x >> kMedBits) == p0) d0 = dg;
                            if ((x >> kMedBits) == p1) d1 = dg;
                        }
                        const unsigned m0 = __match_any_sync(0xffffffffu, d0);
                        if (d0 != 0xffffffffu && (__ffs(m0) - 1) == lane) atomicAdd(&hist[0][d0], __popc(m0));
                        if (first) continue;  // both order statistics share the first digit's histogram
                        const unsigned m1 = __match_any_sync(0xffffffffu, d1);
                        if (d1 != 0xffffffffu && (__ffs(m1) - 1) == lane) atomicAdd(&hist[1][d1], __popc(m1));
                    }
                }
            }
            if (first) {  // the count of the rank's complete-instance deltas comes with the first pass
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                if (lane == 0 && c) atomicAdd(&s_cnt, c);
            }
            __syncthreads();
            const unsigned long long cnt = s_cnt;
            if (cnt == 0) break;
            // digit of each order statistic: a block scan over the bins (two per thread)
            const unsigned long long k0 = first ? (cnt - 1) / 2 : s_k[0], k1 = first ? cnt / 2 : s_k[1];
            const unsigned* h1 = hist[first ? 0 : 1];
            const unsigned a0 = hist[0][2 * threadIdx.x], b0 = hist[0][2 * threadIdx.x + 1];
            const unsigned a1 = h1[2 * threadIdx.x], b1 = h1[2 * threadIdx.x + 1];
            unsigned e0, e1;
            med_scan2(a0 + b0, a1 + b1, e0, e1, s_ws);
            if (k0 >= e0 && k0 < e0 + a0 + b0) {
                const bool lo = k0 < e0 + a0;
                s_pref[0] |= (unsigned long long)(2 * threadIdx.x + (lo ? 0 : 1)) << sh;
                s_k[0] = k0 - e0 - (lo ? 0 : a0);
            }
            if (k1 >= e1 && k1 < e1 + a1 + b1) {
                const bool lo = k1 < e1 + a1;
                s_pref[1] |= (unsigned long long)(2 * threadIdx.x + (lo ? 0 : 1)) << sh;
                s_k[1] = k1 - e1 - (lo ? 0 : a1);
            }
            first = false;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const unsigned long long cnt = s_cnt;
            if (cnt == 0) {
                has_off[r] = 0;
                off[r] = 0;
            } else {
                const int64_t lo = int64_t(s_pref[0]) + dmin, hi = int64_t(s_pref[1]) + dmin;
                has_off[r] = 1;
                off[r] = cnt % 2 ? hi : (lo + hi) / 2;
                atomicAdd(n_total, cnt);
            }
        }
        __syncthreads();
    }
}


// Windowing (bundle.cpp:270-279): max aligned exit per complete instance, init 0.
__global__ void k_coll_aligned_exit(uint64_t n, const uint64_t* key, const uint32_t* inst_of,
                                    const int64_t* s_exit, const unsigned* inst_ingroup, unsigned n_group,
                                    const int64_t* off, unsigned long long* inst_aexit, uint64_t rmask) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
         p += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t g = inst_of[p];
        if (inst_ingroup[g] < n_group) continue;
        uint32_t r = uint32_t(key[p] & rmask);
        atomicMax((long long*)&inst_aexit[g], (long long)(s_exit[p] - off[r]));
    }
}

__global__ void k_coll_window_select(uint64_t n_inst, const unsigned* inst_ingroup, unsigned n_group,
                                     const unsigned long long* inst_aexit, int64_t ws, uint64_t* wkey,
                                     uint32_t* winst, unsigned long long* n_out) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < n_inst;
         g += uint64_t(gridDim.x) * blockDim.x) {
        if (inst_ingroup[g] < n_group) continue;
        long long mx = (long long)inst_aexit[g];
        if (mx < ws) continue;
        unsigned long long o = atomicAdd(n_out, 1ull);
        wkey[o] = uint64_t(mx) ^ 0x8000000000000000ull;  // order-preserving
        winst[o] = uint32_t(g);
    }
}

__global__ void k_coll_winv(uint64_t n_w, const uint32_t* winst_sorted, uint32_t* inst_w) {
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < n_w;
         w += uint64_t(gridDim.x) * blockDim.x)
        inst_w[winst_sorted[w]] = uint32_t(w);
}

// entry_lateness (collective.cpp:127-142): adj = entry - off, min, (adj-min)/1e6.
__global__ void k_coll_minadj(uint64_t n, const uint64_t* key, const uint32_t* inst_of, const uint32_t* inst_w,
                              const int64_t* s_entry, const int64_t* off, long long* wmin, uint64_t rmask) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
         p += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t w = inst_w[inst_of[p]];
        if (w == 0xffffffffu) continue;
        uint32_t r = uint32_t(key[p] & rmask);
        atomicMin(&wmin[w], (long long)(s_entry[p] - off[r]));
    }
}

__global__ void k_coll_lateness(uint64_t n, const uint64_t* key, const uint32_t* inst_of,
                                const uint32_t* inst_w, const int64_t* s_entry, const int64_t* off,
                                const long long* wmin, uint64_t n_w, double* lat /* [rank_span][n_w] */, uint64_t rmask) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
         p += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t w = inst_w[inst_of[p]];
        if (w == 0xffffffffu) continue;
        uint32_t r = uint32_t(key[p] & rmask);
        int64_t adj = s_entry[p] - off[r];
        lat[uint64_t(r) * n_w + w] = __ddiv_rn(__ll2double_rn(adj - wmin[w]), 1e6);
    }
}

__global__ void k_coll_itertimes(uint64_t n_w, const uint64_t* wkey_sorted, double* it) {
    for (uint64_t w = 1 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < n_w;
         w += uint64_t(gridDim.x) * blockDim.x) {
        long long a = (long long)(wkey_sorted[w] ^ 0x8000000000000000ull);
        long long b = (long long)(wkey_sorted[w - 1] ^ 0x8000000000000000ull);
        it[w - 1] = __ddiv_rn(__ll2double_rn(a - b), 1e6);
    }
}

// Per rank: flags, mean lateness (alert: over >=2-rank instances; median
// reference: over all), mean z over flagged — each summed in instance order
// (diagnosis.cpp:97-110, bit-exact: the same sequence of double roundings).
// One warp per rank, in chunks of kStragChunk instances: all lanes load the
// chunk (coalesced row of the rank-major matrix), decide presence / alert /
// flag and z, and stage (value, z, bits) in shared memory; then lanes 0, 1, 2
// run the three in-order add chains side by side over the chunk (lane 0: all
// present, lane 1: present in >= 2-rank instances, lane 2: z of flagged), one
// dependent add per element per chain and no shuffles.
constexpr int kStragChunk = 128;
constexpr int kStragWarps = 8;
constexpr int kStragPer = kStragChunk / 32;
__global__ void __launch_bounds__(kStragWarps * 32) k_straggler_rank(
    uint64_t n_w, int r_lo, int r_hi, const double* lat, double k, const double* mu_w, const double* sigma_w,
    const uint32_t* m_w, uint8_t* present, double* mean_all, double* mean_alert, double* z_mean, uint64_t* flags,
    uint8_t* has_z) {
    __shared__ double s_val[kStragWarps][kStragChunk];
    __shared__ double s_z[kStragWarps][kStragChunk];
    __shared__ uint8_t s_bits[kStragWarps][kStragChunk];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int r = r_lo + int((blockIdx.x * blockDim.x + threadIdx.x) >> 5); r < r_hi;
         r += int((gridDim.x * blockDim.x) >> 5)) {
        double acc = 0.0;  // lane 0: Σ all present, lane 1: Σ alert, lane 2: Σ z of flagged
        uint64_t n_all = 0, n2 = 0, nz = 0;
        const double* row = lat + uint64_t(r) * n_w;
        // chunk c's row values and instance statistics are loaded into registers
        // before chunk c-1's add chains run, so the loads are in flight meanwhile
        double l_n[kStragPer], mu_n[kStragPer], sg_n[kStragPer];
        uint32_t m_n[kStragPer];
        auto fetch = [&](uint64_t c0) {
#pragma unroll
            for (int u = 0; u < kStragPer; ++u) {
                const uint64_t w = c0 + u * 32 + lane;
                const bool in = w < n_w;
                l_n[u] = in ? row[w] : nan("");
                m_n[u] = in ? m_w[w] : 0u;
                mu_n[u] = in ? mu_w[w] : 0.0;
                sg_n[u] = in ? sigma_w[w] : 0.0;
            }
        };
        uint32_t cn_prev = 0;
        if (n_w) fetch(0);
        for (uint64_t c0 = 0; c0 < n_w + kStragChunk; c0 += kStragChunk) {
            const bool have = c0 < n_w;
            const uint32_t cn = have ? uint32_t(n_w - c0 < kStragChunk ? n_w - c0 : kStragChunk) : 0;
            double lv[kStragPer], zv[kStragPer];
            uint8_t bits[kStragPer];
            if (have) {  // decide presence / alert / flag and z of chunk c (registers)
#pragma unroll
                for (int u = 0; u < kStragPer; ++u) {
                    const double l = l_n[u];
                    const bool two = m_n[u] >= 2;
                    bool fl = false;
                    double z = 0.0;
                    if (l == l && two) {
                        const double mu = mu_n[u], sg = sg_n[u];
                        fl = sg > 0.0 && l > __dadd_rn(mu, __dmul_rn(k, sg));
                        if (fl) z = __ddiv_rn(__dsub_rn(l, mu), sg);
                    }
                    const bool pres = l == l;
                    n_all += __popc(__ballot_sync(0xffffffffu, pres));
                    n2 += __popc(__ballot_sync(0xffffffffu, pres && two));
                    nz += __popc(__ballot_sync(0xffffffffu, fl));
                    lv[u] = l;
                    zv[u] = z;
                    bits[u] = uint8_t((pres ? 1 : 0) | (pres && two ? 2 : 0) | (fl ? 4 : 0));
                }
                if (c0 + kStragChunk < n_w) fetch(c0 + kStragChunk);
            }
            // chains of chunk c-1 (staged in shared memory by the previous step)
            if (cn_prev && lane < 3) {
                const double* src = lane == 2 ? s_z[wid] : s_val[wid];
#pragma unroll 8
                for (uint32_t j = 0; j < cn_prev; ++j) {
                    const double v = src[j];
                    if ((s_bits[wid][j] >> lane) & 1) acc = __dadd_rn(acc, v);
                }
            }
            __syncwarp();
            if (have) {
#pragma unroll
                for (int u = 0; u < kStragPer; ++u) {
                    s_val[wid][u * 32 + lane] = lv[u];
                    s_z[wid][u * 32 + lane] = zv[u];
                    s_bits[wid][u * 32 + lane] = (u * 32 + lane) < int(cn) ? bits[u] : 0;
                }
            }
            __syncwarp();
            cn_prev = cn;
        }
        const double s_all = __shfl_sync(0xffffffffu, acc, 0);
        const double s2 = __shfl_sync(0xffffffffu, acc, 1);
        const double sz = __shfl_sync(0xffffffffu, acc, 2);
        if (lane == 0) {
            present[r] = n_all > 0;
            mean_all[r] = n_all ? __ddiv_rn(s_all, double(n_all)) : 0.0;
            mean_alert[r] = n2 ? __ddiv_rn(s2, double(n2)) : 0.0;
            z_mean[r] = nz ? __ddiv_rn(sz, double(nz)) : 0.0;
            flags[r] = nz;
            has_z[r] = nz > 0;
        }
    }
}

// ------------------------------------------- regular streams, column form
// When every stream is regular (instance k of a stream = the k-th event of each
// of its ranks), the per-instance reductions are column reductions over the
// stream's [rank][k] event matrix: one thread per (k, chunk of up to kColChunk
// rank segments) reads its column with coalesced loads (consecutive k are
// adjacent in every segment), reduces in registers and issues one atomic per
// chunk; ranks and instances are implicit (no per-event key or instance id).
constexpr uint32_t kColChunk = 64;
struct ColItems {
    const uint64_t* off;   // [M+1] prefix of the items' k counts
    const uint32_t* j0;    // [M] first segment of the chunk
    const uint32_t* j1;    // [M] end segment
    const uint64_t* ib;    // [M] instance id of k = 0
    uint32_t M;
    uint64_t total;
};
__device__ __forceinline__ bool col_item(const ColItems& c, uint64_t t, uint32_t& m, uint32_t& k) {
    if (t >= c.total) return false;
    uint32_t lo = 0, hi = c.M - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (c.off[mid] <= t) lo = mid; else hi = mid - 1;
    }
    m = lo;
    k = uint32_t(t - c.off[lo]);
    return true;
}
__global__ void k_col_inst(ColItems c, const uint32_t* seg_pos, const uint32_t* seg_rank, const int64_t* s_exit,
                           const uint8_t* member, unsigned long long* imax, unsigned* iing) {
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < c.total; t += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t m, k;
        col_item(c, t, m, k);
        long long mx = LLONG_MIN;
        unsigned ing = 0;
#pragma unroll 4
        for (uint32_t j = c.j0[m]; j < c.j1[m]; ++j) {
            mx = max(mx, (long long)s_exit[seg_pos[j] + k]);
            ing += member[seg_rank[j]];
        }
        const uint64_t g = c.ib[m] + k;
        atomicMax((long long*)&imax[g], mx);
        if (ing) atomicAdd(&iing[g], ing);
    }
}
__global__ void k_col_deltas(ColItems c, const uint32_t* seg_pos, const int64_t* s_exit,
                             const unsigned long long* imax, const unsigned* iing, unsigned n_group, int64_t* dval,
                             long long* dmin) {
    long long lo = 0;
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < c.total; t += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t m, k;
        col_item(c, t, m, k);
        const uint64_t g = c.ib[m] + k;
        const bool ok = iing[g] >= n_group;
        const long long mx = (long long)imax[g];
#pragma unroll 4
        for (uint32_t j = c.j0[m]; j < c.j1[m]; ++j) {
            const uint64_t p = seg_pos[j] + k;
            const int64_t d = ok ? s_exit[p] - mx : 1;
            dval[p] = d;
            if (ok) lo = min(lo, (long long)d);
        }
    }
    for (int o = 16; o > 0; o >>= 1) lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    if ((threadIdx.x & 31) == 0) atomicMin(dmin, lo);
}
__global__ void k_col_aligned_exit(ColItems c, const uint32_t* seg_pos, const uint32_t* seg_rank, const int64_t* s_exit,
                                   const unsigned* iing, unsigned n_group, const int64_t* off,
                                   unsigned long long* aexit) {
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < c.total; t += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t m, k;
        col_item(c, t, m, k);
        const uint64_t g = c.ib[m] + k;
        if (iing[g] < n_group) continue;
        long long mx = LLONG_MIN;
#pragma unroll 4
        for (uint32_t j = c.j0[m]; j < c.j1[m]; ++j) mx = max(mx, (long long)(s_exit[seg_pos[j] + k] - off[seg_rank[j]]));
        atomicMax((long long*)&aexit[g], mx);
    }
}
__global__ void k_col_minadj(ColItems c, const uint32_t* seg_pos, const uint32_t* seg_rank, const int64_t* s_entry,
                             const uint32_t* inst_w, const int64_t* off, long long* wmin) {
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < c.total; t += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t m, k;
        col_item(c, t, m, k);
        const uint32_t w = inst_w[c.ib[m] + k];
        if (w == 0xffffffffu) continue;
        long long mn = LLONG_MAX;
#pragma unroll 4
        for (uint32_t j = c.j0[m]; j < c.j1[m]; ++j) mn = min(mn, (long long)(s_entry[seg_pos[j] + k] - off[seg_rank[j]]));
        atomicMin(&wmin[w], mn);
    }
}
__global__ void k_col_lateness(ColItems c, const uint32_t* seg_pos, const uint32_t* seg_rank, const int64_t* s_entry,
                               const uint32_t* inst_w, const int64_t* off, const long long* wmin, uint64_t n_w,
                               double* lat) {
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < c.total; t += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t m, k;
        col_item(c, t, m, k);
        const uint32_t w = inst_w[c.ib[m] + k];
        if (w == 0xffffffffu) continue;
        const long long base = wmin[w];
#pragma unroll 4
        for (uint32_t j = c.j0[m]; j < c.j1[m]; ++j) {
            const uint32_t r = seg_rank[j];
            lat[uint64_t(r) * n_w + w] = __ddiv_rn(__ll2double_rn(s_entry[seg_pos[j] + k] - off[r] - base), 1e6);
        }
    }
}

// ------------------------------------------------ rank-sharded stage d
// When the collective events are sharded by rank over the GPUs of one group
// (stg_window.shard_streams & STG_SHARD_COLL), each GPU runs the kernels above
// on its own ranks' (stream, rank) segments; what crosses GPUs are the
// per-stream and per-instance partials below (reduced / gathered over NCCL).

// Per local stream: min first entry, min / max per-rank event count, written
// at the stream's global index (each global stream is at most one local one).
__global__ void k_coll_stream_stats(int n_streams, const uint32_t* st_seg, const uint32_t* seg_pos,
                                    const int64_t* s_entry, const uint32_t* lg, uint32_t n_gs, long long* min_first,
                                    uint32_t* kk /* [0, n_gs): kmax, [n_gs, 2 n_gs): ~kmin */) {
    const int s = blockIdx.x;
    if (s >= n_streams) return;
    const uint32_t a = st_seg[s], b = st_seg[s + 1];
    __shared__ long long s_min;
    __shared__ unsigned s_kmin, s_kmax;
    if (threadIdx.x == 0) {
        s_min = LLONG_MAX;
        s_kmin = 0xffffffffu;
        s_kmax = 0;
    }
    __syncthreads();
    for (uint32_t j = a + threadIdx.x; j < b; j += blockDim.x) {
        atomicMin(&s_min, (long long)s_entry[seg_pos[j]]);
        const uint32_t len = seg_pos[j + 1] - seg_pos[j];
        atomicMin(&s_kmin, len);
        atomicMax(&s_kmax, len);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t g = lg[s];
        min_first[g] = s_min;
        kk[g] = s_kmax;
        kk[n_gs + g] = ~s_kmin;
    }
}

// coarse pre-alignment of each local segment against the group-wide first entry
__global__ void k_coll_coarse(uint64_t n_seg, const uint32_t* seg_pos, const uint32_t* seg_stream, const uint32_t* lg,
                              const int64_t* s_entry, const long long* min_first, int64_t* coarse) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < n_seg; j += uint64_t(gridDim.x) * blockDim.x)
        coarse[j] = s_entry[seg_pos[j]] - min_first[lg[seg_stream[j]]];
}

// Work item t of the local regular proof -> (local stream, k); lk_base over
// local streams is the prefix sum of the streams' global min counts.
__device__ __forceinline__ int local_stream_of(const uint64_t* lk_base, int n_streams, uint64_t t) {
    int lo = 0, hi = n_streams - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (lk_base[mid] <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Seed candidate of instance (stream, k) from this GPU's ranks: the lowest
// pre-aligned entry (ties to the lowest rank) and that event's exit.  Candidates
// of all GPUs are gathered; the seed is the first minimum in world-rank order,
// which is the lowest rank because the shards are ascending rank intervals.
__global__ void k_coll_seed_cand(int n_streams, const uint32_t* st_seg, const uint32_t* seg_pos,
                                 const int64_t* coarse, const int64_t* s_entry, const int64_t* s_exit,
                                 const uint64_t* lk_base, uint64_t n_k, const uint32_t* lg, const uint64_t* k_base,
                                 long long* cand /* [K][2] */) {
    const int lane = threadIdx.x & 31;
    for (uint64_t t = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; t < n_k;
         t += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const int s = local_stream_of(lk_base, n_streams, t);
        const uint32_t k = uint32_t(t - lk_base[s]);
        const uint32_t a = st_seg[s], b = st_seg[s + 1];
        long long best = LLONG_MAX;
        uint32_t bj = 0xffffffffu;
        for (uint32_t j = a + lane; j < b; j += 32) {
            const long long e = s_entry[seg_pos[j] + k] - coarse[j];
            if (e < best) {
                best = e;
                bj = j;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long ob = __shfl_xor_sync(0xffffffffu, best, o);
            const uint32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (ob < best || (ob == best && oj < bj)) {
                best = ob;
                bj = oj;
            }
        }
        if (lane == 0) {
            const uint64_t gi = k_base[lg[s]] + k;
            cand[2 * gi] = best;
            cand[2 * gi + 1] = s_exit[seg_pos[bj] + k] - coarse[bj];
        }
    }
}

// The regular-case proof on this GPU's heads against the group-wide seed.
__global__ void k_coll_regular_sh(int n_streams, const uint32_t* st_seg, const uint32_t* seg_pos,
                                  const int64_t* coarse, const int64_t* s_entry, const int64_t* s_exit,
                                  const uint64_t* lk_base, uint64_t n_k, const uint32_t* lg, const uint64_t* k_base,
                                  uint64_t K, const long long* cand_all, int world, int64_t skew,
                                  uint32_t* first_fail /* global stream index */) {
    const int lane = threadIdx.x & 31;
    for (uint64_t t = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; t < n_k;
         t += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const int s = local_stream_of(lk_base, n_streams, t);
        const uint32_t k = uint32_t(t - lk_base[s]);
        const uint64_t gi = k_base[lg[s]] + k;
        long long best = LLONG_MAX, best_exit = 0;
        for (int q = 0; q < world; ++q) {  // first minimum in world order
            const long long e = cand_all[(uint64_t(q) * K + gi) * 2];
            if (e < best) {
                best = e;
                best_exit = cand_all[(uint64_t(q) * K + gi) * 2 + 1];
            }
        }
        const uint32_t a = st_seg[s], b = st_seg[s + 1];
        bool ok = true;
        for (uint32_t j = a + lane; j < b && ok; j += 32) {
            const uint64_t p = seg_pos[j] + k;
            const long long e = s_entry[p] - coarse[j], x = s_exit[p] - coarse[j];
            ok = e <= best_exit + skew && x + skew >= best;
        }
        ok = __all_sync(0xffffffffu, ok);
        if (!ok && lane == 0) atomicMin(first_fail + lg[s], k);
    }
}

// detect_straggler's per-instance sums (diagnosis.cpp:82-96) split along the
// rank order: each GPU continues the chains of the GPUs before it over its
// own ranks [r0, r1) — the same sequence of double roundings as one pass over
// all ranks.  Pass 1: (Σ l, count) per instance; pass 2: Σ (l - μ)².
__global__ void k_strag_chain1(uint64_t n_w, int r0, int r1, const double* lat, double* chain /* [n_w][2] */) {
    const int lane = threadIdx.x & 31;
    for (uint64_t w = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; w < n_w;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        double acc = chain[2 * w];
        uint32_t m = 0;
        for (int rb = r0; rb < r1; rb += 32) {
            const int r = rb + lane;
            const double l = r < r1 ? lat[uint64_t(r) * n_w + w] : nan("");
            const unsigned pres = __ballot_sync(0xffffffffu, l == l);
            m += __popc(pres);
            for (unsigned q = pres; q; q &= q - 1) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, l, __ffs(q) - 1));
        }
        if (lane == 0) {
            chain[2 * w] = acc;
            chain[2 * w + 1] += double(m);
        }
    }
}
__global__ void k_strag_mu(uint64_t n_w, const double* chain, double* mu_w, uint32_t* m_w) {
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < n_w; w += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t m = uint32_t(chain[2 * w + 1]);
        m_w[w] = m;
        mu_w[w] = m >= 2 ? __ddiv_rn(chain[2 * w], double(m)) : 0.0;
    }
}
__global__ void k_strag_chain2(uint64_t n_w, int r0, int r1, const double* lat, const double* mu_w,
                               const uint32_t* m_w, double* s2_w) {
    const int lane = threadIdx.x & 31;
    for (uint64_t w = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; w < n_w;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        if (m_w[w] < 2) continue;
        const double mu = mu_w[w];
        double s2 = s2_w[w];
        for (int rb = r0; rb < r1; rb += 32) {
            const int r = rb + lane;
            const double l = r < r1 ? lat[uint64_t(r) * n_w + w] : nan("");
            const double d = __dsub_rn(l, mu);
            const double dd = __dmul_rn(d, d);
            for (unsigned q = __ballot_sync(0xffffffffu, l == l); q; q &= q - 1)
                s2 = __dadd_rn(s2, __shfl_sync(0xffffffffu, dd, __ffs(q) - 1));
        }
        if (lane == 0) s2_w[w] = s2;
    }
}
__global__ void k_strag_sigma(uint64_t n_w, const double* s2_w, const uint32_t* m_w, double* sigma_w) {
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < n_w; w += uint64_t(gridDim.x) * blockDim.x)
        if (m_w[w] >= 2) sigma_w[w] = __dsqrt_rn(__ddiv_rn(s2_w[w], double(m_w[w])));
}
// The same chains with one thread per instance, for many instances (C4:
// 50k): the warp's 32 instances are adjacent in each rank row, so every step
// of the rank loop is one coalesced 256 B read; the chain stays in the thread.
constexpr int kChainU = 8;
__global__ void k_strag_chain1_t(uint64_t n_w, int r0, int r1, const double* lat, double* chain) {
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < n_w; w += uint64_t(gridDim.x) * blockDim.x) {
        double acc = chain[2 * w];
        uint32_t m = 0;
        int r = r0;
        for (; r + kChainU <= r1; r += kChainU) {
            double v[kChainU];
#pragma unroll
            for (int u = 0; u < kChainU; ++u) v[u] = __ldcs(lat + uint64_t(r + u) * n_w + w);
#pragma unroll
            for (int u = 0; u < kChainU; ++u)
                if (v[u] == v[u]) {
                    acc = __dadd_rn(acc, v[u]);
                    ++m;
                }
        }
        for (; r < r1; ++r) {
            const double l = lat[uint64_t(r) * n_w + w];
            if (l == l) {
                acc = __dadd_rn(acc, l);
                ++m;
            }
        }
        chain[2 * w] = acc;
        chain[2 * w + 1] += double(m);
    }
}
__global__ void k_strag_chain2_t(uint64_t n_w, int r0, int r1, const double* lat, const double* mu_w,
                                 const uint32_t* m_w, double* s2_w) {
    for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < n_w; w += uint64_t(gridDim.x) * blockDim.x) {
        if (m_w[w] < 2) continue;
        const double mu = mu_w[w];
        double s2 = s2_w[w];
        int r = r0;
        for (; r + kChainU <= r1; r += kChainU) {
            double v[kChainU];
#pragma unroll
            for (int u = 0; u < kChainU; ++u) v[u] = __ldcs(lat + uint64_t(r + u) * n_w + w);
#pragma unroll
            for (int u = 0; u < kChainU; ++u)
                if (v[u] == v[u]) {
                    const double d = __dsub_rn(v[u], mu);
                    s2 = __dadd_rn(s2, __dmul_rn(d, d));
                }
        }
        for (; r < r1; ++r) {
            const double l = lat[uint64_t(r) * n_w + w];
            if (l == l) {
                const double d = __dsub_rn(l, mu);
                s2 = __dadd_rn(s2, __dmul_rn(d, d));
            }
        }
        s2_w[w] = s2;
    }
}

// local stream keys (group, kind) for the global stream union
__global__ void k_stream_keys(const unsigned long long* counts, const uint32_t* st_pos, const uint64_t* key, int rbits,
                              uint64_t* skey) {
    const uint64_t n_st = counts[1];
    for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < n_st; s += uint64_t(gridDim.x) * blockDim.x)
        skey[s] = key[st_pos[s]] >> rbits;
}

__global__ void k_fill_f64(double* p, uint64_t n, double v) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}
__global__ void k_fill_i64(long long* p, uint64_t n, long long v) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}
__global__ void k_iota(uint32_t* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = uint32_t(i);
}
__global__ void k_max_rank(uint64_t n, const int32_t* r, int* mx, int* mn) {
    int a = -1, b = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        a = max(a, r[i]);
        b = min(b, r[i]);
    }
    atomicMax(mx, a);
    atomicMin(mn, b);
}

// flag = 1 unless the events' ranks are non-decreasing in input order (the
// common rank-major layout): then a stable sort on the stream bits alone
// already yields (stream, rank, input order)
__global__ void k_rank_unsorted(uint64_t n, const int32_t* r, int* flag) {
    for (uint64_t i = 1 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        if (r[i] < r[i - 1]) *flag = 1;
}

// ================================================================ gpu / os
// build_group_data GPU loop (bundle.cpp:302-306)
__global__ void k_gpu_sums(uint64_t n, const int32_t* rank, const uint32_t* kern, const int64_t* start,
                           const int64_t* dur, const int64_t* off, int64_t ws, uint32_t n_kern,
                           unsigned long long* sums, uint8_t* present, int* err) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        int r = rank[i];
        uint32_t k = kern[i];
        if (k >= n_kern) {
            *err = 1;
            continue;
        }
        if (start[i] - off[r] < ws) continue;
        atomicAdd(&sums[uint64_t(r) * n_kern + k], (unsigned long long)dur[i]);
        present[uint64_t(r) * n_kern + k] = 1;
    }
}

// build_group_data OS loop (bundle.cpp:308-320)
__global__ void k_os_sums(uint64_t n, const int32_t* rank, const int64_t* wstart, const int64_t* p50,
                          const int64_t* p99, const int64_t* mig, const uint64_t* irq_off,
                          const uint32_t* irq_key, const int64_t* irq_val, const uint64_t* sirq_off,
                          const uint32_t* sirq_key, const int64_t* sirq_val, const int64_t* off, int64_t ws,
                          uint32_t n_keys, unsigned long long* irq, uint8_t* irq_p, unsigned long long* sirq,
                          uint8_t* sirq_p, long long* p50m, long long* p99m, unsigned long long* migs,
                          uint8_t* present, int* err) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        int r = rank[i];
        if (wstart[i] - off[r] + 5000000000ll < ws) continue;
        present[r] = 1;
        for (uint64_t k = irq_off[i]; k < irq_off[i + 1]; ++k) {
            uint32_t key = irq_key[k];
            if (key >= n_keys) { *err = 1; continue; }
            atomicAdd(&irq[uint64_t(r) * n_keys + key], (unsigned long long)irq_val[k]);
            irq_p[uint64_t(r) * n_keys + key] = 1;
        }
        for (uint64_t k = sirq_off[i]; k < sirq_off[i + 1]; ++k) {
            uint32_t key = sirq_key[k];
            if (key >= n_keys) { *err = 1; continue; }
            atomicAdd(&sirq[uint64_t(r) * n_keys + key], (unsigned long long)sirq_val[k]);
            sirq_p[uint64_t(r) * n_keys + key] = 1;
        }
        atomicMax(&p50m[r], (long long)p50[i]);
        atomicMax(&p99m[r], (long long)p99[i]);
        atomicAdd(&migs[r], (unsigned long long)mig[i]);
    }
}

// ===================================================== samples: stage a+b
struct AggParams {
    const int64_t* ts;
    const uint64_t* foff;
    const uint64_t* pc;
    const uint16_t* bin;
    const uint64_t* rank_soff;   // [R+1]
    const int64_t* rank_clk;     // [R] clock offset of each CPU rank
    const uint8_t* active;       // [R]
    int R;
    int64_t ws;
    const DevTable* tabs;
    uint32_t n_bins;
    int mode;
    AggSlot* slots;
    const uint64_t* tab_off;     // [R] slot offset
    const uint32_t* tab_mask;    // [R]
    unsigned* tab_used;
    int* tab_overflow;
    PfxSlot* pfx;                // prefix cache (raw non-leaf chain -> symbolized terms)
    uint32_t pfx_mask;
    UnkSet unk;
    unsigned long long* n_in;    // [R]
    int* unsorted;               // [R]
    unsigned long long* err_empty;  // [R] min rank-relative index
    int* err_bin;
    unsigned long long* stat;    // [0] prefix hits, [1] misses
    uint64_t n_samples;
    uint64_t n_frames;
    uint64_t salt;               // fingerprint key of this attempt (0 = default)
    int use_pfx;                 // 0: no prefix cache (verification retry)
    int weak_pfx;                // tests: 4-bit prefix-cache keys (forced collisions)
};

// atom.global.cas.b128 against an empty (0, 0) key: returns the previous key.
__device__ __forceinline__ void cas128(unsigned long long* addr, unsigned long long va, unsigned long long vb,
                                       unsigned long long& oa, unsigned long long& ob) {
    asm volatile("{\n\t.reg .b128 c, v, d;\n\t"
                 "mov.b128 c, {%2, %2};\n\t"
                 "mov.b128 v, {%3, %4};\n\t"
                 "atom.global.cas.b128 d, [%5], c, v;\n\t"
                 "mov.b128 {%0, %1}, d;\n\t}"
                 : "=l"(oa), "=l"(ob)
                 : "l"(0ull), "l"(va), "l"(vb), "l"(addr)
                 : "memory");
}

// Open addressing on the 128-bit key (hi, lo): one 16 B L2 read per probe; an
// empty slot is claimed with a single 128-bit CAS (both halves at once, so no
// reader ever sees a half-written key and no fence is needed); counts and the
// per-rank occupancy are fire-and-forget reductions (the host compares the
// occupancy with the 50 % load limit after the kernel and retries larger); a
// probe run longer than kMaxProbe also marks the table for a retry.  rep is
// read only after the kernel.
constexpr uint32_t kMaxProbe = 512;
__device__ __forceinline__ uint32_t agg_insert(AggSlot* T, uint32_t mask, uint64_t fa, uint64_t fb, uint32_t rep,
                                               uint32_t cnt, unsigned* used, int* overflow) {
    uint32_t i = uint32_t(fb >> 20) & mask;
    for (uint32_t probe = 0; probe <= mask && probe < kMaxProbe; ++probe) {
        ulonglong2 cur = __ldcg(reinterpret_cast<const ulonglong2*>(T + i));  // (hi, lo) in one L2 read
        if ((cur.x | cur.y) == 0) {
            unsigned long long oa, ob;
            cas128(&T[i].hi, fa, fb, oa, ob);
            if ((oa | ob) == 0) {
                T[i].rep = rep;
                if (cnt) atomicAdd(&T[i].count, cnt);
                atomicAdd(used, 1u);
                return i;
            }
            cur.x = oa;
            cur.y = ob;
        }
        if (cur.x == fa && cur.y == fb) {
            if (cnt) atomicAdd(&T[i].count, cnt);
            return i;
        }
        i = (i + 1) & mask;
    }
    *overflow = 1;
    return 0xffffffffu;
}

// Raw-chain fingerprint, block form.  Frames are taken in aligned blocks of 8
// (the vector loads' granularity); a block contributes five 64x64->128-bit
// products — four over pc pairs, one over the packed bins — each operand
// xor-keyed by its slot, the block's position q and the run's salt.  Each
// product also adds its operands linearly (the other half gets the partner), so
// no operand value annihilates its partner: with y fixed, x -> (x*y + y,
// mulhi(x, y) + x) changes whenever x does (for y = 0 the high half still
// moves by x), and symmetrically for y.  The sums (ha, hb) with the sample's
// alignment and depth mixed in at the end are the prefix-cache key; frames
// outside the sample's non-leaf range are zeroed, so the key depends on the
// chain, its depth and f0 mod 8 only.  A run with verification on re-checks
// every sample against a direct symbolization and retries with a new salt and
// no cache on a mismatch (Runner::samples).
__device__ __forceinline__ void mum_acc(uint64_t x, uint64_t y, uint64_t& ha, uint64_t& hb) {
    ha += x * y + y;
    hb += __umul64hi(x, y) + x;
}
__device__ __forceinline__ void raw_block(const uint64_t (&pc)[8], uint64_t b01, uint64_t b23, uint64_t q,
                                          uint64_t salt, uint64_t& ha, uint64_t& hb) {
    const uint64_t B = ((q + 1) * 0x9e3779b97f4a7c15ull) ^ salt;
    mum_acc(pc[0] ^ B ^ 0x243f6a8885a308d3ull, pc[1] ^ B ^ 0x13198a2e03707344ull, ha, hb);
    mum_acc(pc[2] ^ B ^ 0xa4093822299f31d0ull, pc[3] ^ B ^ 0x082efa98ec4e6c89ull, ha, hb);
    mum_acc(pc[4] ^ B ^ 0x452821e638d01377ull, pc[5] ^ B ^ 0xbe5466cf34e90c6cull, ha, hb);
    mum_acc(pc[6] ^ B ^ 0xc0ac29b7c97c50ddull, pc[7] ^ B ^ 0x3f84d5b5b5470917ull, ha, hb);
    mum_acc(b01 ^ B ^ 0x9216d5d98979fb1bull, b23 ^ B ^ 0xd1310ba698dfb5acull, ha, hb);
}

// 256-bit read-only global load (sm_100: LDG.E.ENL2.256), 32-byte aligned.
__device__ __forceinline__ void ld256(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
}

// One aligned block of 8 frames for this lane: pcs by two 256-bit loads (each
// lane takes a whole 32 B sector per instruction, read-only path, no L1
// allocation), bins by one 16 B load; scalar and zero-filled past the end of
// the frame array.  PF == 1 adds the L2::256B prefetch-size hint.
template <int PF>
__device__ __forceinline__ void load_block(const uint64_t* pc, const uint16_t* bin, uint64_t n_frames, uint64_t bb,
                                           uint64_t (&pcs)[8], uint4& bq) {
    if (bb + 8 <= n_frames) {
        if (PF == 1) {
            asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u64 {%0, %1, %2, %3}, [%4];"
                         : "=l"(pcs[0]), "=l"(pcs[1]), "=l"(pcs[2]), "=l"(pcs[3]) : "l"(pc + bb));
            asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u64 {%0, %1, %2, %3}, [%4];"
                         : "=l"(pcs[4]), "=l"(pcs[5]), "=l"(pcs[6]), "=l"(pcs[7]) : "l"(pc + bb + 4));
            asm volatile("ld.global.nc.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(bq.x), "=r"(bq.y), "=r"(bq.z), "=r"(bq.w) : "l"(bin + bb));
        } else {
            ld256(pc + bb, pcs[0], pcs[1], pcs[2], pcs[3]);
            ld256(pc + bb + 4, pcs[4], pcs[5], pcs[6], pcs[7]);
            bq = __ldg(reinterpret_cast<const uint4*>(bin + bb));
        }
    } else {
        uint32_t bw[4] = {0, 0, 0, 0};
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const bool ok = bb + t < n_frames;
            pcs[t] = ok ? pc[bb + t] : 0;
            bw[t >> 1] |= (ok ? uint32_t(bin[bb + t]) : 0u) << (16 * (t & 1));
        }
        bq = make_uint4(bw[0], bw[1], bw[2], bw[3]);
    }
}

// The same aligned block as a pure stream read: whole blocks only, read-only
// path without L1 allocation, and an L2 evict-first policy so that the ~80 GB
// frame stream does not push the aggregation tables, the prefix cache and the
// symbol tables out of L2.
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void load_block_stream(const uint64_t* pc, const uint16_t* bin, uint64_t bb, uint64_t pol,
                                                  uint64_t (&pcs)[8], uint4& bq) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=l"(pcs[0]), "=l"(pcs[1]), "=l"(pcs[2]), "=l"(pcs[3]) : "l"(pc + bb), "l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=l"(pcs[4]), "=l"(pcs[5]), "=l"(pcs[6]), "=l"(pcs[7]) : "l"(pc + bb + 4), "l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(bq.x), "=r"(bq.y), "=r"(bq.z), "=r"(bq.w) : "l"(bin + bb), "l"(pol));
}

// Prefix cache.  Entries are immutable once published: the writer claims the
// 128-bit key (hi, lo) with one CAS, then stores (ta, tb) as one 16 B store.  A
// reader takes (hi, lo) and (ta, tb) with two 16-byte L2 reads issued together;
// a key seen with (ta, tb) still zero (racing the writer) is treated as a miss.
__device__ __forceinline__ void pfx_put(PfxSlot* T, uint32_t mask, uint64_t ha, uint64_t hb, uint64_t ta, uint64_t tb) {
    uint32_t i = uint32_t(hb >> 24) & mask;
    for (int probe = 0; probe < 16; ++probe) {
        unsigned long long oa, ob;
        cas128(&T[i].hi, ha, hb, oa, ob);
        if ((oa | ob) == 0) {
            __stcg(reinterpret_cast<ulonglong2*>(&T[i].ta), make_ulonglong2(ta, tb));
            return;
        }
        if (oa == ha && ob == hb) return;  // someone else stores the same chain
        i = (i + 1) & mask;
    }
}

__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
    const uint32_t sa = uint32_t(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
}


// The fused hot kernel (stage a+b), one lane per sample.  A warp takes 32
// consecutive samples — one contiguous block of frames in HBM — and owns a
// contiguous range of such batches, so its rank only moves forward:
//  phase 0  lane s loads its ts and CSR bound (coalesced; the neighbours' by
//           shuffle), applies the window filter on the aligned clock
//           (bundle.cpp:290-294);
//  phase 1  lane s streams its own frames in aligned blocks of 8 (two 256-bit
//           pc loads + 16 B of bins) and folds the NON-LEAF frames into a
//           128-bit raw-chain fingerprint (raw_block); the warp as a whole
//           reads its 20 KB block sector-complete;
//  phase 2  lane s: prefix-cache probe (the raw chain's symbolized terms —
//           return addresses repeat, so hits dominate) overlapped with the leaf
//           lookup in the staged table (symfile.cpp:54-75), fingerprint of the
//           root-first name sequence, and one insert into the rank's
//           open-addressing table with __match_any pre-aggregation;
//  misses   the warp symbolizes the missing chains cooperatively and fills
//           the cache.
template <bool SMEM_TABS, int MINB, int UB, int UBC, bool COOP = true>
__global__ void __launch_bounds__(kThreads, MINB) k_sym_agg(AggParams p) {
    __shared__ DevTable s_tabs[kMaxSmemBins];
    if (SMEM_TABS) {
        for (uint32_t i = threadIdx.x; i < p.n_bins; i += blockDim.x) s_tabs[i] = p.tabs[i];
        __syncthreads();
    }
    __shared__ ulonglong4 s_acc[kThreads / 32][32];  // cooperative phase 1: (Σa, Σb, leaf pc, leaf bin) per sample
    const DevTable* tabs = SMEM_TABS ? s_tabs : p.tabs;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t n_batches = (p.n_samples + 31) / 32;
    const uint64_t pol = evict_first_policy();
    unsigned hits = 0, misses = 0;  // lane 0's per-warp tallies (< 2^32 per warp)
    // batch order: contiguous ranges per warp, so a warp's rank only moves
    // forward and advances by compares instead of a search per batch
    const uint64_t per = (n_batches + nwarps - 1) / nwarps;
    const uint64_t b_begin = warp * per;
    const uint64_t b_end = b_begin + per < n_batches ? b_begin + per : n_batches;
    const uint64_t b_step = 1;
    int r_cur = 0;
    if (b_begin < b_end) {
        const uint64_t q = b_begin * 32;
        int lo = 0, hi = p.R - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (__ldg(p.rank_soff + mid) <= q) lo = mid; else hi = mid - 1;
        }
        r_cur = lo;
    }
    // phase-0 stream values of the next batch, copied one batch ahead into
    // shared memory with asynchronous copies (in flight while the current batch
    // streams its frames and runs its lookups, and holding no registers)
    __shared__ uint64_t s_nx[kThreads / 32][4][32];  // ts, frame offset, next frame offset, previous ts
    uint64_t* nxw = &s_nx[threadIdx.x >> 5][0][0];
    auto load0 = [&](uint64_t b) {
        const uint64_t i = b * 32 + lane;
        const uint64_t q = i < p.n_samples ? i : p.n_samples - 1;
        cp_async8(nxw + lane, p.ts + q);
        cp_async8(nxw + 32 + lane, p.foff + q);
        if (lane == 31 || i + 1 >= p.n_samples) cp_async8(nxw + 64 + lane, p.foff + q + 1);
        if (lane == 0 && q > 0) cp_async8(nxw + 96, p.ts + q - 1);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (b_begin < b_end) load0(b_begin);
    for (uint64_t bt = b_begin; bt < b_end; bt += b_step) {
        // ---------------- phase 0: lane s owns sample i; its stream values were
        // loaded during the previous batch, the next batch's are issued now
        const uint64_t i = bt * 32 + lane;
        const bool valid = i < p.n_samples;
        const uint64_t q = valid ? i : p.n_samples - 1;
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        const int64_t t = int64_t(nxw[lane]);
        uint64_t f0 = nxw[32 + lane];
        const bool own_next = lane == 31 || i + 1 >= p.n_samples;
        uint64_t f1 = own_next ? nxw[64 + lane] : 0;
        const int64_t t_prev = lane == 0 && q > 0 ? int64_t(nxw[96]) : 0;
        __syncwarp();
        if (bt + b_step < b_end) load0(bt + b_step);
        int r = r_cur;
        while (q >= __ldg(p.rank_soff + r + 1)) ++r;
        r_cur = __shfl_sync(0xffffffffu, r, 31);
        const uint64_t rs = __ldg(p.rank_soff + r);
        {
            const uint64_t up = __shfl_down_sync(0xffffffffu, f0, 1);
            if (!own_next) f1 = up;
            int64_t tp = __shfl_up_sync(0xffffffffu, t, 1);
            if (lane == 0) tp = t_prev;
            if (valid && q > rs && t < tp && p.active[r]) p.unsorted[r] = 1;
        }
        bool inwin = valid && p.active[r] && t - __ldg(p.rank_clk + r) >= p.ws;
        if (inwin && f1 == f0) {
            atomicMin(p.err_empty + r, (unsigned long long)(i - rs));
            inwin = false;
        }
        if (!inwin) f0 = f1 = 0;
        const uint32_t depth = uint32_t(f1 - f0);
        uint64_t leaf_pc = 0, ha = 0, hb = 0;
        uint32_t leaf_bin = 0;
        // ---------------- phase 1, cooperative form: when the 32 samples are all
        // in the window, equally deep (D = 8·NB, NB a power of two <= 32) and
        // block-aligned, the warp streams its contiguous frame range with
        // coalesced loads — lane l takes block l of every 256-frame step (2 KB of
        // pcs + 512 B of bins per warp instruction triple) — computes that
        // block's raw_block term, sums the NB terms of each sample with a
        // butterfly over its lane group, and the group's first lane (which also
        // holds the leaf frame) hands (Σa, Σb, leaf) to the sample's own lane
        // through shared memory.  Same terms, same sums as the per-lane form.
        bool coop = false;
        {
            const uint64_t A = __shfl_sync(0xffffffffu, f0, 0);
            const uint32_t d0 = __shfl_sync(0xffffffffu, depth, 0);
            const uint32_t nb = d0 >> 3;
            coop = COOP && __all_sync(0xffffffffu, inwin && depth == d0) && d0 >= 8 && (d0 & 7) == 0 &&
                   (A & 7) == 0 && nb <= 32 && (nb & (nb - 1)) == 0;
            if (COOP && coop) {
                const int lg = __ffs(nb) - 1;
                const int wid = threadIdx.x >> 5;
                // UBC steps per round trip: all their loads are issued before any hashing
                for (uint32_t it0 = 0; it0 < nb; it0 += UBC) {
                    uint64_t pcs[UBC][8];
                    uint4 bq[UBC];
#pragma unroll
                    for (int u = 0; u < UBC; ++u)
                        if (u == 0 || it0 + u < nb)
                            load_block_stream(p.pc, p.bin, A + 8ull * ((it0 + u) * 32 + lane), pol, pcs[u], bq[u]);
#pragma unroll
                    for (int u = 0; u < UBC; ++u) {
                        if (u > 0 && it0 + u >= nb) break;
                        const uint32_t g = (it0 + u) * 32 + lane;
                        const uint32_t qb = g & (nb - 1);
                        const uint64_t lpc = pcs[u][0];
                        const uint32_t lbin = bq[u].x & 0xffffu;
                        if (qb == 0) {  // the leaf is not part of the chain
                            pcs[u][0] = 0;
                            bq[u].x &= 0xffff0000u;
                        }
                        uint64_t xa = 0, xb = 0;
                        raw_block(pcs[u], uint64_t(bq[u].x) | (uint64_t(bq[u].y) << 32),
                                  uint64_t(bq[u].z) | (uint64_t(bq[u].w) << 32), qb, p.salt, xa, xb);
                        for (uint32_t o = 1; o < nb; o <<= 1) {
                            xa += __shfl_xor_sync(0xffffffffu, xa, o);
                            xb += __shfl_xor_sync(0xffffffffu, xb, o);
                        }
                        if (qb == 0) s_acc[wid][g >> lg] = make_ulonglong4(xa, xb, lpc, lbin);
                    }
                }
                __syncwarp();
                const ulonglong4 v = s_acc[wid][lane];
                ha = v.x;
                hb = v.y;
                leaf_pc = v.z;
                leaf_bin = uint32_t(v.w);
                __syncwarp();
            }
        }
        // ---------------- phase 1, per-lane form: this lane's frames, 8 per step
        if (inwin && !coop) {
            const uint64_t a0 = f0 & ~7ull;
            for (uint64_t bs = a0; bs < f1; bs += 8 * UB) {
                // UB blocks per step: all their loads are issued before any hashing
                constexpr int NB = UB;
                uint64_t pcs[NB][8];
                uint4 bq[NB];
#pragma unroll
                for (int u = 0; u < NB; ++u)
                    if (u == 0 || bs + 8 * u < f1) load_block<0>(p.pc, p.bin, p.n_frames, bs + 8 * u, pcs[u], bq[u]);
#pragma unroll
                for (int u = 0; u < NB; ++u) {
                    const uint64_t bb = bs + 8 * u;
                    if (u > 0 && bb >= f1) break;
                    if (!(bb > f0 && bb + 8 <= f1)) {  // boundary block: take the leaf, zero the rest
                        uint32_t bw[4] = {bq[u].x, bq[u].y, bq[u].z, bq[u].w};
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            const uint64_t j = bb + t;
                            const uint32_t bv = (bw[t >> 1] >> (16 * (t & 1))) & 0xffffu;
                            if (j == f0) {
                                leaf_pc = pcs[u][t];
                                leaf_bin = bv;
                            }
                            if (!(j > f0 && j < f1)) {
                                pcs[u][t] = 0;
                                bw[t >> 1] &= ~(0xffffu << (16 * (t & 1)));
                            }
                        }
                        bq[u] = make_uint4(bw[0], bw[1], bw[2], bw[3]);
                    }
                    raw_block(pcs[u], uint64_t(bq[u].x) | (uint64_t(bq[u].y) << 32),
                              uint64_t(bq[u].z) | (uint64_t(bq[u].w) << 32), (bb - a0) >> 3, p.salt, ha, hb);
                }
            }
        }
        const unsigned need = __ballot_sync(0xffffffffu, inwin && depth > 1);
        const uint64_t shape = uint64_t(depth) | (uint64_t(f0 & 7) << 32);
        uint64_t my_ra = mix_a(ha ^ (shape * 0x8cb92ba72f3d8dd7ull));
        uint64_t my_rb = mix_b(hb + shape);
        if (my_ra == 0) my_ra = 1;
        if (my_rb == 0) my_rb = 1;
        if (p.weak_pfx) {  // tests only (stg_config.debug_weak_prefix_key)
            my_ra = 1 + (my_ra & 3);
            my_rb = 1 + (my_rb & 3);
        }
        // ---------------- phase 2: per-lane cache probe overlapped with the leaf lookup
        const bool want_pfx = inwin && depth > 1 && p.use_pfx;
        // issue the first probe of both structures before either resolves
        const uint32_t pslot = uint32_t(my_rb >> 24) & p.pfx_mask;
        ulonglong2 pa = make_ulonglong2(0, 0), pb = make_ulonglong2(0, 0);
        if (want_pfx) {
            pa = __ldcg(reinterpret_cast<const ulonglong2*>(p.pfx + pslot));
            pb = __ldcg(reinterpret_cast<const ulonglong2*>(p.pfx + pslot) + 1);
        }
        uint32_t leaf_key = kUnknownBit;
        bool leaf_search = false;
        uint32_t blo = 0, bhi = 0;
        const DevTable* T = nullptr;
        if (inwin) {
            if (leaf_bin < p.n_bins) {
                T = tabs + leaf_bin;
                if (T->valid && leaf_pc >= T->base) {
                    const uint64_t bk = (leaf_pc - T->base) >> T->shift;
                    if (bk >= T->nb) {
                        blo = bhi = T->n - 1;
                    } else {
                        blo = __ldg(T->bucket + bk);
                        bhi = __ldg(T->bucket + bk + 1);
                    }
                    leaf_search = true;
                }
            } else {
                *p.err_bin = 1;
            }
        }
        uint64_t ta = 0, tb = 0;
        bool hit = !(inwin && depth > 1);
        if (want_pfx) {
            uint32_t slot = pslot;
            for (int probe = 0; probe < 16; ++probe) {
                if (pa.x == 0) break;
                if (pa.x == my_ra) {
                    if (pa.y == my_rb && (pb.x | pb.y) != 0) {
                        ta = pb.x;
                        tb = pb.y;
                        hit = true;
                    }
                    if (pa.y == my_rb || pa.y == 0) break;
                }
                slot = (slot + 1) & p.pfx_mask;
                pa = __ldcg(reinterpret_cast<const ulonglong2*>(p.pfx + slot));
                pb = __ldcg(reinterpret_cast<const ulonglong2*>(p.pfx + slot) + 1);
            }
        }
        if (leaf_search) {
            // bisection down to <= 2 candidates (the bucket index usually leaves
            // 1-2), then both candidates' entries in one round trip: the answer is
            // the last whose start is <= pc (symfile.cpp:54-75)
            while (bhi - blo > 1) {
                const uint32_t mid = (blo + bhi + 1) >> 1;
                if (__ldg(&T->e[mid].x) <= leaf_pc) blo = mid; else bhi = mid - 1;
            }
            ulonglong2 e = __ldg(T->e + blo);
            const ulonglong2 e1 = blo < bhi ? __ldg(T->e + bhi) : e;
            if (blo < bhi && e1.x <= leaf_pc) e = e1;
            if (p.mode == STG_LOOKUP_NEAREST_LOWER) {
                leaf_key = uint32_t(e.y >> 32);
            } else {
                const uint32_t size = uint32_t(e.y);
                const bool in = size == 0 ? leaf_pc == e.x : leaf_pc < e.x + uint64_t(size);
                if (in) leaf_key = uint32_t(e.y >> 32);
            }
        }
        if (inwin && leaf_key == kUnknownBit) leaf_key = kUnknownBit | unk_get(p.unk, leaf_bin, leaf_pc);
        unsigned miss = __ballot_sync(0xffffffffu, !hit);
        hits += __popc(need & ~miss) * (lane == 0);
        misses += __popc(miss) * (lane == 0);
        while (miss) {
            const int src = __ffs(miss) - 1;
            miss &= miss - 1;
            const uint64_t a0 = __shfl_sync(0xffffffffu, f0, src);
            const uint64_t a1 = __shfl_sync(0xffffffffu, f1, src);
            const uint64_t d = a1 - a0;
            uint64_t xa = 0, xb = 0;
            for (uint64_t j = a0 + 1 + lane; j < a1; j += 32) {
                uint32_t key = resolve_frame(tabs, p.n_bins, p.pc[j], p.bin[j], p.mode, p.unk, p.err_bin);
                uint32_t pos = uint32_t(d - 1 - (j - a0));  // root-first position
                xa += term_a(key, pos, p.salt);
                xb += term_b(key, pos, p.salt);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                xa += __shfl_xor_sync(0xffffffffu, xa, o);
                xb += __shfl_xor_sync(0xffffffffu, xb, o);
            }
            if (lane == src) {
                ta = xa;
                tb = xb;
                if (p.use_pfx) pfx_put(p.pfx, p.pfx_mask, my_ra, my_rb, ta, tb);
            }
        }
        uint64_t fa = 0, fb = 0;
        if (inwin) {
            ta += term_a(leaf_key, depth - 1, p.salt);
            tb += term_b(leaf_key, depth - 1, p.salt);
            fp_finish(ta, tb, depth, fa, fb);
        }
        // ---------------- aggregate: identical (rank, stack) in the batch combine
        const unsigned act = __ballot_sync(0xffffffffu, inwin);
        if (act) {
            const unsigned mr = __match_any_sync(0xffffffffu, r) & act;
            const unsigned m = __match_any_sync(0xffffffffu, inwin ? fa : 0ull) & mr;
            if (inwin && (__ffs(m) - 1) == lane) {
                agg_insert(p.slots + __ldg(p.tab_off + r), __ldg(p.tab_mask + r), fa, fb, uint32_t(i - rs),
                               __popc(m), p.tab_used + r, p.tab_overflow + r);
            }
            if (inwin && (__ffs(mr) - 1) == lane) atomicAdd(p.n_in + r, (unsigned long long)__popc(mr));
        }
    }
    if (lane == 0 && (hits | misses)) {
        atomicAdd(p.stat, (unsigned long long)hits);
        atomicAdd(p.stat + 1, (unsigned long long)misses);
    }
}

// ------------------------------------------------------------ verification
// stg_config.verify: the full compare of aggregate_samples (samples.cpp:67-76)
// for the fused kernel.  One warp per sample: the sample is symbolized again
// frame by frame (no prefix cache), its sequence fingerprint recomputed and
// looked up in its rank's table (read-only, the insert's probe order), and its
// names compared one by one with the slot's representative sample; each
// sample then adds 1 to its slot's recount.  Any miss or difference (a
// fingerprint collision somewhere) is counted in *bad.
__device__ __forceinline__ bool same_frame(uint32_t a, uint32_t b, const UnkSlot* unk, const uint32_t* bin_canon) {
    if (a == b) return true;
    if (!(a & b & kUnknownBit)) return false;  // real names: equal keys <=> equal names
    // two unknown slots name the same label iff (build id, offset) agree
    const UnkSlot x = unk[a & ~kUnknownBit], y = unk[b & ~kUnknownBit];
    return x.pc == y.pc && bin_canon[x.bin1 - 1] == bin_canon[y.bin1 - 1];
}
__global__ void k_sym_verify(AggParams p, const uint32_t* bin_canon, unsigned* vcount, unsigned long long* bad) {
    __shared__ DevTable s_tabs[kMaxSmemBins];
    for (uint32_t i = threadIdx.x; i < p.n_bins && i < kMaxSmemBins; i += blockDim.x) s_tabs[i] = p.tabs[i];
    __syncthreads();
    const DevTable* tabs = p.n_bins <= kMaxSmemBins ? s_tabs : p.tabs;
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    unsigned long long n_bad = 0;
    for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < p.n_samples; i += nw) {
        int lo = 0, hi = p.R - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (p.rank_soff[mid] <= i) lo = mid; else hi = mid - 1;
        }
        const int r = lo;
        const uint64_t f0 = p.foff[i], f1 = p.foff[i + 1];
        if (!p.active[r] || p.ts[i] - p.rank_clk[r] < p.ws || f1 == f0) continue;
        const uint64_t d = f1 - f0;
        uint64_t xa = 0, xb = 0;
        for (uint64_t pos = lane; pos < d; pos += 32) {
            const uint64_t j = f1 - 1 - pos;
            const uint32_t key = resolve_frame(tabs, p.n_bins, p.pc[j], p.bin[j], p.mode, p.unk, p.err_bin);
            xa += term_a(key, uint32_t(pos), p.salt);
            xb += term_b(key, uint32_t(pos), p.salt);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            xa += __shfl_xor_sync(0xffffffffu, xa, o);
            xb += __shfl_xor_sync(0xffffffffu, xb, o);
        }
        uint64_t fa, fb;
        fp_finish(xa, xb, d, fa, fb);
        const AggSlot* T = p.slots + p.tab_off[r];
        const uint32_t mask = p.tab_mask[r];
        uint32_t k = uint32_t(fb >> 20) & mask;
        bool found = false;
        for (uint32_t probe = 0; probe <= mask && probe < kMaxProbe; ++probe) {
            const ulonglong2 cur = *reinterpret_cast<const ulonglong2*>(T + k);
            if ((cur.x | cur.y) == 0) break;
            if (cur.x == fa && cur.y == fb) {
                found = true;
                break;
            }
            k = (k + 1) & mask;
        }
        bool ok = found;
        if (found) {
            const uint64_t rep = p.rank_soff[r] + T[k].rep;
            const uint64_t g0 = p.foff[rep], g1 = p.foff[rep + 1];
            ok = g1 - g0 == d;
            for (uint64_t pos = lane; ok && pos < d; pos += 32) {
                const uint32_t a = resolve_frame(tabs, p.n_bins, p.pc[f1 - 1 - pos], p.bin[f1 - 1 - pos], p.mode,
                                                 p.unk, p.err_bin);
                const uint32_t b = resolve_frame(tabs, p.n_bins, p.pc[g1 - 1 - pos], p.bin[g1 - 1 - pos], p.mode,
                                                 p.unk, p.err_bin);
                if (!same_frame(a, b, p.unk.slots, bin_canon)) ok = false;
            }
            ok = __all_sync(0xffffffffu, ok);
            if (lane == 0) atomicAdd(vcount + p.tab_off[r] + k, 1u);
        }
        if (!ok) ++n_bad;
    }
    if (lane == 0 && n_bad) atomicAdd(bad, n_bad);
}

// Every slot's recount must equal its count (no sample lost or double counted).
__global__ void k_count_check(uint64_t n_slots, const AggSlot* slots, const unsigned* vcount, unsigned long long* bad) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_slots; i += uint64_t(gridDim.x) * blockDim.x)
        if ((slots[i].hi | slots[i].lo) != 0 && slots[i].count != vcount[i]) atomicAdd(bad, 1ull);
}

// Cross-rank sequence dedupe (k_seq_dedupe merges lines on the 128-bit
// fingerprint): every line's representative must spell the same names as its
// sequence's representative.  Warp per line.
__global__ void k_line_verify(uint64_t L, const uint64_t* l_rep, const uint32_t* l_gid, const uint64_t* seq_rep,
                              const uint64_t* foff, const uint64_t* pc, const uint16_t* bin, const DevTable* tabs_g,
                              uint32_t n_bins, int mode, UnkSet unk, int* err_bin, const uint32_t* bin_canon,
                              unsigned long long* bad) {
    __shared__ DevTable s_tabs[kMaxSmemBins];
    for (uint32_t i = threadIdx.x; i < n_bins && i < kMaxSmemBins; i += blockDim.x) s_tabs[i] = tabs_g[i];
    __syncthreads();
    const DevTable* tabs = n_bins <= kMaxSmemBins ? s_tabs : tabs_g;
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t l = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; l < L; l += nw) {
        const uint64_t a = l_rep[l], b = seq_rep[l_gid[l]];
        if (a == b) continue;
        const uint64_t a0 = foff[a], a1 = foff[a + 1], b0 = foff[b], b1 = foff[b + 1];
        bool ok = a1 - a0 == b1 - b0;
        for (uint64_t pos = lane; ok && pos < a1 - a0; pos += 32) {
            const uint32_t x = resolve_frame(tabs, n_bins, pc[a1 - 1 - pos], bin[a1 - 1 - pos], mode, unk, err_bin);
            const uint32_t y = resolve_frame(tabs, n_bins, pc[b1 - 1 - pos], bin[b1 - 1 - pos], mode, unk, err_bin);
            if (!same_frame(x, y, unk.slots, bin_canon)) ok = false;
        }
        ok = __all_sync(0xffffffffu, ok);
        if (!ok && lane == 0) atomicAdd(bad, 1ull);
    }
}

// Rare path: exact in-window timestamp regression check for ranks whose full
// stream is not sorted (aggregate_samples samples.cpp:55-58 sees only the
// in-window subsequence).  One thread per flagged rank.
__global__ void k_regress_exact(int n, const int* ranks, const uint64_t* rank_soff, const int64_t* ts,
                                const int64_t* clk, int64_t ws, unsigned long long* out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    int r = ranks[t];
    bool have = false;
    int64_t prev = 0;
    unsigned long long res = ~0ull;
    for (uint64_t i = rank_soff[r]; i < rank_soff[r + 1]; ++i) {
        int64_t v = ts[i];
        if (v - clk[r] < ws) continue;
        if (have && v < prev) {
            res = i - rank_soff[r];
            break;
        }
        have = true;
        prev = v;
    }
    out[t] = res;
}

// ======================================================= fold: lines, seqs
__global__ void k_compact_lines(int R, const uint64_t* tab_off, const uint32_t* tab_mask, const AggSlot* slots,
                                const uint64_t* rank_soff, uint32_t* l_rank, uint64_t* l_hi, uint64_t* l_lo,
                                uint32_t* l_count, uint64_t* l_rep, unsigned long long* n_out) {
    // one output reservation per block (block-wide ballot counts), not per line
    __shared__ unsigned warp_n[kThreads / 32];
    __shared__ unsigned long long base;
    const int r = blockIdx.y;
    const uint32_t cap = tab_mask[r] + 1;
    const AggSlot* T = slots + tab_off[r];
    const uint64_t soff = rank_soff[r];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < cap; i0 += gridDim.x * blockDim.x) {
        const uint32_t i = i0 + threadIdx.x;
        AggSlot s{};
        if (i < cap) s = T[i];
        const bool live = s.hi != 0;
        const unsigned m = __ballot_sync(0xffffffffu, live);
        if (lane == 0) warp_n[wid] = __popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned tot = 0;
            for (int w = 0; w < kThreads / 32; ++w) {
                const unsigned c = warp_n[w];
                warp_n[w] = tot;
                tot += c;
            }
            base = tot ? atomicAdd(n_out, (unsigned long long)tot) : 0;
        }
        __syncthreads();
        if (live) {
            const unsigned long long o = base + warp_n[wid] + __popc(m & ((1u << lane) - 1));
            l_rank[o] = uint32_t(r);
            l_hi[o] = s.hi;
            l_lo[o] = s.lo;
            l_count[o] = s.count;
            l_rep[o] = soff + s.rep;
        }
        __syncthreads();
    }
}

// Global dedupe of symbolized stacks across ranks: fingerprint -> sequence id.
// stat = {distinct count (u32) | overflow (u32) << 32, Σ lengths, max length}: the
// host reads all three with one download.
__global__ void k_seq_dedupe(uint64_t L, const uint64_t* l_hi, const uint64_t* l_lo, const uint64_t* l_rep,
                             SeqSlot* T, uint64_t mask, unsigned long long* stat, uint32_t* l_gid, uint64_t* seq_rep,
                             const uint64_t* foff) {
    unsigned* n_seq = reinterpret_cast<unsigned*>(stat);
    int* overflow = reinterpret_cast<int*>(stat) + 1;
    for (uint64_t l = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; l < L; l += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t fa = l_hi[l], fb = l_lo[l];
        uint64_t i = mix_a(fa ^ fb) & mask;
        uint32_t gid = 0xffffffffu;
        // a table sized from the previous window may be too small: past half
        // load, or after a long probe run, the call retries at 2 slots per line
        for (uint64_t probe = 0; probe <= mask && probe < 1024; ++probe) {
            unsigned long long cur = *(volatile unsigned long long*)&T[i].hi;
            if (cur == 0) {
                cur = atomicCAS(&T[i].hi, 0ull, (unsigned long long)fa);
                if (cur == 0) {
                    gid = atomicAdd(n_seq, 1u);
                    if (uint64_t(gid) + 1 > (mask + 1) / 2) *overflow = 1;
                    T[i].lo = fb;
                    const uint64_t rep = l_rep[l];
                    T[i].rep = rep;
                    seq_rep[gid] = rep;
                    const unsigned long long len = foff[rep + 1] - foff[rep];
                    atomicAdd(stat + 1, len);
                    atomicMax(stat + 2, len);
                    __threadfence();
                    atomicExch(&T[i].gid, gid);
                    break;
                }
            }
            if (cur == fa) {
                unsigned g;
                while ((g = *(volatile unsigned*)&T[i].gid) == 0xffffffffu) __nanosleep(16);
                __threadfence();
                if (*(volatile unsigned long long*)&T[i].lo == fb) {
                    gid = g;
                    break;
                }
            }
            i = (i + 1) & mask;
        }
        if (gid == 0xffffffffu) *overflow = 1;
        l_gid[l] = gid;
    }
}

// Re-symbolize each distinct stack's representative sample into the arena,
// root first (folded.cpp:24-26).  Warp per sequence.
__global__ void k_seq_materialize(uint32_t G, const uint64_t* seq_rep, const uint64_t* seq_off,
                                  const uint64_t* foff, const uint64_t* pc, const uint16_t* bin,
                                  const DevTable* tabs_g, uint32_t n_bins, int mode, UnkSet unk, int* err_bin,
                                  uint32_t* arena) {
    __shared__ DevTable s_tabs[kMaxSmemBins];
    for (uint32_t i = threadIdx.x; i < n_bins && i < kMaxSmemBins; i += blockDim.x) s_tabs[i] = tabs_g[i];
    __syncthreads();
    const DevTable* tabs = n_bins <= kMaxSmemBins ? s_tabs : tabs_g;
    const int lane = threadIdx.x & 31;
    for (uint64_t g = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; g < G;
         g += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        uint64_t s = seq_rep[g];
        uint64_t f0 = foff[s], f1 = foff[s + 1];
        uint64_t d = f1 - f0;
        uint32_t* out = arena + seq_off[g];
        for (uint64_t pos = lane; pos < d; pos += 32) {
            uint64_t j = f1 - 1 - pos;
            out[pos] = resolve_frame(tabs, n_bins, pc[j], bin[j], mode, unk, err_bin);
        }
    }
}

// Distinct unresolved frames as packed {pc, slot | bin << 32} records (one download).
__global__ void k_unk_compact(uint32_t cap, const UnkSlot* slots, ulonglong2* out, unsigned* n_out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x) {
        uint32_t b = slots[i].bin1;
        if (b == 0 || b == 0xffffffffu) continue;
        unsigned o = atomicAdd(n_out, 1u);
        out[o] = make_ulonglong2(slots[i].pc, uint64_t(i) | (uint64_t(b - 1) << 32));
    }
}

// Final name rank: real name i -> i + #{unknown labels < name i}; unknown slot ->
// its label's merged rank (host-computed).
// pos_sorted holds, for every distinct label that is not itself a real name, the
// number of real names below it; a real name i therefore moves up by
// upper_bound(pos_sorted, i).
__device__ __forceinline__ uint32_t remap_key(uint32_t e, const uint32_t* unk_final, const uint32_t* pos_sorted,
                                              uint32_t n_pos) {
    if (e & kUnknownBit) return unk_final[e & ~kUnknownBit];
    uint32_t lo = 0, hi = n_pos;  // upper_bound(pos_sorted, e)
    while (lo < hi) {
        uint32_t m = (lo + hi) >> 1;
        if (pos_sorted[m] <= e) lo = m + 1; else hi = m;
    }
    return e + lo;
}

__global__ void k_remap(uint64_t n, uint32_t* arena, const uint32_t* unk_final, const uint32_t* pos_sorted,
                        uint32_t n_pos) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        arena[i] = remap_key(arena[i], unk_final, pos_sorted, n_pos);
}

__global__ void k_fill_gid(SeqSlot* s, uint64_t n) {  // empty slot: key 0, gid unpublished
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        reinterpret_cast<ulonglong4*>(s)[i] = make_ulonglong4(0ull, 0ull, 0xffffffffull, 0ull);
    }
}
__global__ void k_seq_len64(uint32_t G, const uint64_t* seq_rep, const uint64_t* foff, uint64_t* len) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < G; g += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t s = seq_rep[g];
        len[g] = foff[s + 1] - foff[s];
    }
}
__global__ void k_dense_final(uint64_t n, const uint32_t* used, const uint32_t* used_scan, uint32_t* dense_final) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        if (used[i]) dense_final[used_scan[i]] = uint32_t(i);
}
// symbolize verb: frame-wise keys (resolve_stacks symrepo.cpp:122-143)
__global__ void k_resolve(uint64_t n, const uint64_t* pc, const uint16_t* bin, const DevTable* tabs_g,
                          uint32_t n_bins, int mode, UnkSet unk, int* err_bin, uint32_t* out) {
    __shared__ DevTable s_tabs[kMaxSmemBins];
    for (uint32_t i = threadIdx.x; i < n_bins && i < kMaxSmemBins; i += blockDim.x) s_tabs[i] = tabs_g[i];
    __syncthreads();
    const DevTable* tabs = n_bins <= kMaxSmemBins ? s_tabs : tabs_g;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = resolve_frame(tabs, n_bins, pc[i], bin[i], mode, unk, err_bin);
}

// Lexicographic order of name-rank sequences, shorter prefix first — the order
// of std::map<std::vector<std::string>, ...> (folded.cpp:11-19).
struct SeqLess {
    const uint32_t* arena;
    const uint64_t* off;
    __device__ __forceinline__ int cmp(uint32_t a, uint32_t b) const {
        const uint64_t oa = off[a], ob = off[b];
        const uint32_t* x = arena + oa;
        const uint32_t* y = arena + ob;
        const uint64_t la = off[a + 1] - oa, lb = off[b + 1] - ob;
        const uint64_t n = la < lb ? la : lb;
        uint64_t i = 0;
        if (((oa ^ ob) & 3) == 0) {  // same 16-byte phase: compare 4 names per load
            for (; i < n && ((oa + i) & 3); ++i) {
                const uint32_t u = x[i], v = y[i];
                if (u != v) return u < v ? -1 : 1;
            }
            for (; i + 4 <= n; i += 4) {
                const uint4 u = *reinterpret_cast<const uint4*>(x + i);
                const uint4 v = *reinterpret_cast<const uint4*>(y + i);
                if (u.x != v.x) return u.x < v.x ? -1 : 1;
                if (u.y != v.y) return u.y < v.y ? -1 : 1;
                if (u.z != v.z) return u.z < v.z ? -1 : 1;
                if (u.w != v.w) return u.w < v.w ? -1 : 1;
            }
        }
        for (; i < n; ++i) {
            const uint32_t u = x[i], v = y[i];
            if (u != v) return u < v ? -1 : 1;
        }
        return la < lb ? -1 : (la > lb ? 1 : 0);
    }
    __device__ __forceinline__ bool operator()(const uint32_t& a, const uint32_t& b) const { return cmp(a, b) < 0; }
};

__global__ void k_seq_rankflags(uint32_t G, const uint32_t* sorted, SeqLess less, uint32_t* flag) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < G; p += uint64_t(gridDim.x) * blockDim.x)
        flag[p] = p == 0 ? 1u : (less.cmp(sorted[p - 1], sorted[p]) != 0 ? 1u : 0u);
}
__global__ void k_seq_rankset(uint32_t G, const uint32_t* sorted, const uint32_t* incl_scan, uint32_t* seq_rank,
                              uint32_t* dense_rep) {
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < G; p += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t d = incl_scan[p] - 1;
        seq_rank[sorted[p]] = d;
        if (p == 0 || incl_scan[p - 1] != incl_scan[p]) dense_rep[d] = sorted[p];
    }
}

// Sequence order by prefix doubling over aligned blocks: every sequence is
// padded to P = 2^m names with a sentinel (0) below every name (name + 1), so
// comparing padded sequences is exactly the std::map<std::vector<std::string>>
// order (shorter prefix first, folded.cpp:18).  Level k ranks each aligned block
// of 2^k names among all such blocks by the pair of its halves' level-(k-1)
// ranks (a radix sort of 64-bit pair keys); at level m a block is a whole
// sequence, so its rank is the sequence's dense position.
__global__ void k_pd_init(uint64_t n, uint32_t p_log, const uint64_t* off, const uint32_t* arena, uint32_t* cur) {
    for (uint64_t x = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; x < n; x += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t g = x >> p_log, j = x & ((1ull << p_log) - 1);
        const uint64_t o = off[g], len = off[g + 1] - o;
        cur[x] = j < len ? arena[o + j] + 1u : 0u;
    }
}
// key = (left << vb) | right: both values are < 2^vb, so the radix sort runs 2·vb bits
__global__ void k_pd_pairs(uint64_t n, const uint32_t* cur, int vb, uint64_t* key, uint32_t* idx) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint2 v = reinterpret_cast<const uint2*>(cur)[i];
        key[i] = (uint64_t(v.x) << vb) | v.y;
        idx[i] = uint32_t(i);
    }
}
__global__ void k_pd_flags(uint64_t n, const uint64_t* ks, uint32_t* flag) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        flag[i] = (i == 0 || ks[i] != ks[i - 1]) ? 1u : 0u;
}
__global__ void k_pd_scatter(uint64_t n, const uint32_t* idx_s, const uint32_t* rank, uint32_t* cur) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        cur[idx_s[i]] = rank[i];
}
__global__ void k_pd_final(uint32_t G, const uint32_t* cur, uint32_t* seq_rank, uint32_t* dense_rep) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < G; g += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t d = cur[g] - 1;  // ranks are 1-based
        seq_rank[g] = d;
        dense_rep[d] = uint32_t(g);     // any member: equal ranks are equal name sequences
    }
}

__global__ void k_line_keys(uint64_t L, const uint32_t* l_rank, const uint32_t* l_gid, const uint32_t* seq_rank,
                            uint64_t* lkey) {
    for (uint64_t l = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; l < L; l += uint64_t(gridDim.x) * blockDim.x)
        lkey[l] = (uint64_t(l_rank[l]) << 32) | seq_rank[l_gid[l]];
}

__global__ void k_line_bounds(int R, const uint64_t* lkey, uint64_t L, uint64_t* line_off) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= R; r += gridDim.x * blockDim.x) {
        uint64_t key = uint64_t(r) << 32;
        uint64_t a = 0, b = L;
        while (a < b) {
            uint64_t m = (a + b) >> 1;
            if (lkey[m] < key) a = m + 1; else b = m;
        }
        line_off[r] = a;
    }
}

// ============================================================ stage c: diff
// Distinct names of each dense sequence (a name repeated in a stack counts once,
// folded.cpp:49).  Warp per sequence; first pass counts, second writes.
template <bool WRITE>
__global__ void k_seq_distinct(uint32_t S, const uint32_t* dense_rep, const uint64_t* seq_off, const uint32_t* arena,
                               uint32_t* cnt, const uint64_t* dn_off, uint32_t* dn) {
    const int lane = threadIdx.x & 31;
    for (uint64_t s = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; s < S;
         s += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        uint32_t g = dense_rep[s];
        const uint32_t* x = arena + seq_off[g];
        uint64_t d = seq_off[g + 1] - seq_off[g];
        uint32_t base = 0;
        for (uint64_t p0 = 0; p0 < d; p0 += 32) {
            uint64_t p = p0 + lane;
            bool first = false;
            uint32_t v = 0;
            if (p < d) {
                v = x[p];
                first = true;
                for (uint64_t q = 0; q < p; ++q)
                    if (x[q] == v) { first = false; break; }
            }
            unsigned m = __ballot_sync(0xffffffffu, first);
            if (WRITE && first) dn[dn_off[s] + base + __popc(m & ((1u << lane) - 1))] = v;
            base += __popc(m);
        }
        if (!WRITE && lane == 0) cnt[s] = base;
    }
}

// n read on the device (the exclusive sum's last entry): no host round trip
__global__ void k_mark_used(const uint64_t* n_ptr, const uint32_t* dn, uint32_t* used) {
    const uint64_t n = *n_ptr;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        used[dn[i]] = 1;
}
__global__ void k_dense_names(const uint64_t* n_ptr, uint32_t* dn, const uint32_t* used_scan) {
    const uint64_t n = *n_ptr;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        dn[i] = used_scan[dn[i]];  // exclusive scan -> dense index
}

// Inclusive counts per (rank, name), incl[r * F + f] = Σ of the
// counts of rank r's lines whose sequence contains name f (folded.cpp:45-54
// counts a repeated name once per line).  As a sparse product: C[s][r] = the
// count of rank r's line with sequence s (dense S x R, L2-resident), and the
// name -> sequences incidence in column form; a warp walks a slice of the
// column entries, each lane summing 4 ranks of C's row s with one 16-byte load,
// and flushes its per-name partials with one atomic per (name, rank) run.
__global__ void k_lines_to_mat(uint64_t L, const uint64_t* lkey, const unsigned long long* lcount, uint32_t Rp,
                               uint32_t* C) {
    for (uint64_t l = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; l < L; l += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t key = lkey[l];
        C[uint64_t(uint32_t(key)) * Rp + (key >> 32)] = uint32_t(lcount[l]);
    }
}
// (name, sequence) incidence pairs in dn order; sorted by name they form the
// columns of the name x sequence matrix (no atomics on hot names' cursors)
__global__ void k_name_pairs(uint32_t S, const uint64_t* dn_off, const uint32_t* dn, uint32_t* col_f, uint32_t* col_s) {
    const int lane = threadIdx.x & 31;
    for (uint64_t s = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; s < S;
         s += (uint64_t(gridDim.x) * blockDim.x) >> 5)
        for (uint64_t k = dn_off[s] + lane; k < dn_off[s + 1]; k += 32) {
            col_f[k] = dn[k];
            col_s[k] = uint32_t(s);
        }
}
__global__ void k_incl_spmm(const uint64_t* nd_ptr, const uint32_t* col_f, const uint32_t* col_s, const uint32_t* C,
                            uint32_t R, uint32_t Rp, uint64_t F, uint32_t seg, unsigned long long* incl) {
    const uint64_t nd = *nd_ptr;
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t w = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; w * seg < nd; w += nw) {
        const uint64_t e0 = w * seg, e1 = e0 + seg < nd ? e0 + seg : nd;
        for (uint32_t c0 = 0; c0 < R; c0 += 128) {
            const uint32_t r0 = c0 + 4 * lane;
            const bool mine = r0 < Rp;
            unsigned long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            uint32_t cur = col_f[e0];
            auto flush = [&](uint32_t f) {
                if (!mine) return;
                unsigned long long* col = incl + f;
                if (a0 && r0 < R) atomicAdd(col + uint64_t(r0) * F, a0);
                if (a1 && r0 + 1 < R) atomicAdd(col + uint64_t(r0 + 1) * F, a1);
                if (a2 && r0 + 2 < R) atomicAdd(col + uint64_t(r0 + 2) * F, a2);
                if (a3 && r0 + 3 < R) atomicAdd(col + uint64_t(r0 + 3) * F, a3);
                a0 = a1 = a2 = a3 = 0;
            };
            for (uint64_t e = e0; e < e1; ++e) {
                const uint32_t f = col_f[e];
                if (f != cur) {
                    flush(cur);
                    cur = f;
                }
                if (mine) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(C + uint64_t(col_s[e]) * Rp + r0));
                    a0 += v.x;
                    a1 += v.y;
                    a2 += v.z;
                    a3 += v.w;
                }
            }
            flush(cur);
        }
    }
}
// Fallback when the dense S x R count matrix would not fit: warp per line.
__global__ void k_incl_lines(uint64_t L, const uint64_t* lkey, const unsigned long long* lcount, const uint64_t* dn_off,
                             const uint32_t* dn, uint64_t F, unsigned long long* incl) {
    const int lane = threadIdx.x & 31;
    for (uint64_t l = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; l < L;
         l += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const uint64_t key = lkey[l];
        const uint32_t r = uint32_t(key >> 32), s = uint32_t(key);
        const unsigned long long c = lcount[l];
        for (uint64_t k = dn_off[s] + lane; k < dn_off[s + 1]; k += 32) atomicAdd(incl + uint64_t(r) * F + dn[k], c);
    }
}

// compute_waterline (diagnosis.cpp:35-55) per name over the CPU ranks: present
// fractions in rank order then zeros appended, population sigma; flag_ranks
// (:57-71) strictly above mean + k sigma.
// Warp per name: the lanes load 32 ranks' counts and divide in parallel, lane 0
// adds the fractions in rank order (the reference's order), zeros after them.
__device__ __forceinline__ double warp_ordered_sum(double acc, double v, unsigned take) {
    for (unsigned q = take; q; q &= q - 1) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, v, __ffs(q) - 1));
    return acc;
}
__global__ void k_waterline(uint64_t F, const uint32_t* rows, int R, const unsigned long long* incl,
                            const uint64_t* totals, double* mean, double* sd, uint8_t* present_any) {
    const int lane = threadIdx.x & 31;
    for (uint64_t f = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; f < F;
         f += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        double acc = 0.0;
        int np = 0;
        for (int i0 = 0; i0 < R; i0 += 32) {
            const int i = i0 + lane;
            double x = 0.0;
            bool pres = false;
            if (i < R) {
                const uint32_t r = rows[i];
                const unsigned long long c = incl[uint64_t(r) * F + f];
                pres = c != 0;
                if (pres) x = __ddiv_rn(double(c), double(totals[r]));
            }
            const unsigned m = __ballot_sync(0xffffffffu, pres);
            np += __popc(m);
            acc = warp_ordered_sum(acc, x, m);
        }
        const double mu = __ddiv_rn(acc, double(R));
        double s2 = 0.0;
        for (int i0 = 0; i0 < R; i0 += 32) {
            const int i = i0 + lane;
            double dd = 0.0;
            bool pres = false;
            if (i < R) {
                const uint32_t r = rows[i];
                const unsigned long long c = incl[uint64_t(r) * F + f];
                pres = c != 0;
                if (pres) {
                    const double d = __dsub_rn(__ddiv_rn(double(c), double(totals[r])), mu);
                    dd = __dmul_rn(d, d);
                }
            }
            s2 = warp_ordered_sum(s2, dd, __ballot_sync(0xffffffffu, pres));
        }
        if (lane == 0) {
            for (int i = np; i < R; ++i) s2 = __dadd_rn(s2, __dmul_rn(mu, mu));
            present_any[f] = np > 0;
            mean[f] = mu;
            sd[f] = __dsqrt_rn(__ddiv_rn(s2, double(R)));
        }
    }
}

__global__ void k_flag(uint64_t F, const uint32_t* rows, int R, const unsigned long long* incl,
                       const uint64_t* totals, double k, const double* mean, const double* sd, uint32_t* o_r,
                       uint32_t* o_f, double* o_frac, double* o_thr, unsigned long long* n_out,
                       unsigned long long cap) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < F * uint64_t(R);
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t r = rows[i / F], f = i % F;
        unsigned long long c = incl[r * F + f];
        if (!c) continue;
        double fr = __ddiv_rn(double(c), double(totals[r]));
        double thr = __dadd_rn(mean[f], __dmul_rn(k, sd[f]));
        if (fr > thr) {
            unsigned long long o = atomicAdd(n_out, 1ull);
            if (o < cap) {
                o_r[o] = uint32_t(r);
                o_f[o] = uint32_t(f);
                o_frac[o] = fr;
                o_thr[o] = thr;
            }
        }
    }
}

// Per-sequence merged counts for the temporal route (diagnosis.cpp:396-402).
__global__ void k_seq_counts(uint64_t L, const uint64_t* lkey, const unsigned long long* lcount, unsigned long long* sc) {
    for (uint64_t l = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; l < L; l += uint64_t(gridDim.x) * blockDim.x)
        atomicAdd(sc + uint32_t(lkey[l]), lcount[l]);
}

// Hottest path (diagnosis.cpp:184-193 / 413-420): first line in order with the
// strictly greatest count among lines containing dense name f.
// Pass 0: best[0] = max count; pass 1: best[1] = first position with that count.
__global__ void k_hottest(uint64_t n, const uint64_t* seq_of, const unsigned long long* cnt_of, int seq_is_index,
                          const uint64_t* dn_off, const uint32_t* dn, uint32_t f, int pass,
                          unsigned long long* best) {
    // one warp per line: the lanes test 32 of the line's distinct names at once
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n; i += nw) {
        const unsigned long long c = cnt_of[i];
        if (c == 0) continue;
        if (pass == 1 && c != best[0]) continue;
        const uint32_t s = seq_is_index ? uint32_t(i) : uint32_t(seq_of[i]);
        const uint64_t k0 = dn_off[s], k1 = dn_off[s + 1];
        bool has = false;
        for (uint64_t k = k0; k < k1; k += 32) {
            const bool hit = k + lane < k1 && dn[k + lane] == f;
            if (__any_sync(0xffffffffu, hit)) {
                has = true;
                break;
            }
        }
        if (!has || lane != 0) continue;
        if (pass == 0)
            atomicMax(best, c);
        else
            atomicMin(best + 1, (unsigned long long)i);
    }
}

// The hottest line's name sequence, packed for one download: out[0] = found,
// out[1] = length, out[2..] = the names (cap entries at most).
__global__ void k_hot_pack(const unsigned long long* best, const uint64_t* lkey, int merged, const uint32_t* dense_rep,
                           const uint64_t* seq_off, const uint32_t* arena, uint32_t cap, uint32_t* out) {
    const unsigned long long bi = best[1];
    if (bi == ~0ull) {
        if (threadIdx.x == 0) out[0] = out[1] = 0;
        return;
    }
    const uint32_t s = merged ? uint32_t(bi) : uint32_t(lkey[bi]);
    const uint32_t g = dense_rep[s];
    const uint64_t o0 = seq_off[g], len = seq_off[g + 1] - o0;
    if (threadIdx.x == 0) {
        out[0] = 1;
        out[1] = uint32_t(len);
    }
    for (uint64_t k = threadIdx.x; k < len && k < cap; k += blockDim.x) out[2 + k] = arena[o0 + k];
}

// Exact inclusive fractions in the reference's summation order
// (folded.cpp:45-54): (name, line) pairs sorted, then one sequential sum of
// double(count)/double(total) per name in line order.
// want (optional): only names f with want[f] != 0 take part (the diff's
// candidates, see Runner::diagnose); warp per line, lanes over its names.
__global__ void k_pair_count(uint64_t n, uint64_t n0, const uint64_t* lkey0, const uint64_t* lkey1,
                             const uint64_t* dn_off, const uint32_t* dn, const uint8_t* want, uint64_t* cnt) {
    const int lane = threadIdx.x & 31;
    for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n;
         i += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const bool side = i >= n0;
        const uint64_t j = side ? i - n0 : i;
        const uint64_t* lk = side ? lkey1 : lkey0;
        const uint32_t s = lk ? uint32_t(lk[j]) : uint32_t(j);
        const uint64_t k0 = dn_off[s], k1 = dn_off[s + 1];
        uint64_t c = 0;
        if (!want) {
            c = k1 - k0;
        } else {
            for (uint64_t k = k0; k < k1; k += 32)
                c += __popc(__ballot_sync(0xffffffffu, k + lane < k1 && want[dn[k + lane]]));
        }
        if (lane == 0) cnt[i] = c;
    }
}
// Pairs (name, line) of up to two line ranges (side 0: lines [0, n0), side 1:
// [n0, n)); key = (side << NB | name) << LB | line within its side (the stable
// radix sort only runs the NB + 1 side/name bits above LB), value =
// double(count) / double(total of its side).  Warp per line, coalesced.
__global__ void k_pair_emit(uint64_t n, uint64_t n0, const uint64_t* lkey0, const uint64_t* lkey1,
                            const unsigned long long* cnt0, const unsigned long long* cnt1, uint64_t total0,
                            uint64_t total1, const uint64_t* dn_off, const uint32_t* dn, const uint8_t* want,
                            const uint64_t* pair_off, int LB, int NB, uint64_t* keys, double* vals) {
    const double t0 = __ull2double_rn(total0), t1 = __ull2double_rn(total1);
    const int lane = threadIdx.x & 31;
    for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n;
         i += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const bool side = i >= n0;
        const uint64_t j = side ? i - n0 : i;
        const uint64_t* lk = side ? lkey1 : lkey0;
        const uint32_t s = lk ? uint32_t(lk[j]) : uint32_t(j);
        const double x = __ddiv_rn(__ull2double_rn((side ? cnt1 : cnt0)[j]), side ? t1 : t0);  // count / total
        uint64_t o = pair_off[i];
        const uint64_t sb = side ? 1ull << NB : 0ull;
        const uint64_t k0 = dn_off[s], k1 = dn_off[s + 1];
        for (uint64_t kb = k0; kb < k1; kb += 32) {
            const uint64_t k = kb + lane;
            uint32_t f = 0;
            bool ok = k < k1;
            if (ok) {
                f = dn[k];
                if (want) ok = want[f] != 0;
            }
            const unsigned b = __ballot_sync(0xffffffffu, ok);
            if (ok) {
                const uint64_t q = o + __popc(b & ((1u << lane) - 1));
                keys[q] = ((sb | f) << LB) | j;
                vals[q] = x;
            }
            o += __popc(b);
        }
    }
}
// cpu_diff pre-filter (diagnosis.cpp:177-208): a straggler name can pass
// d = fs - fr > delta only if its exact-integer estimate passes delta - margin,
// margin bounding the rounding of the reference's sequential sums (see
// Runner::diagnose); those names alone get the exact line-order sums.
// names of one rank whose own inclusive fraction can exceed lim (a name's
// cpu_diff d = fs - fr <= fs, so only these can pass delta)
__global__ void k_frac_want(uint64_t F, const unsigned long long* row, double total, double lim, uint8_t* want) {
    for (uint64_t f = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; f < F; f += uint64_t(gridDim.x) * blockDim.x) {
        const unsigned long long c = row[f];
        want[f] = c && __ddiv_rn(__ull2double_rn(c), total) > lim;
    }
}
__global__ void k_diff_cands(uint64_t F, const unsigned long long* incl, uint32_t R, uint32_t is, uint32_t iq,
                             double ts, double tr, double lim, uint8_t* want) {
    for (uint64_t f = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; f < F; f += uint64_t(gridDim.x) * blockDim.x) {
        const unsigned long long cs = incl[uint64_t(is) * F + f];
        bool w = false;
        if (cs) {
            const double d = __dsub_rn(__ddiv_rn(__ull2double_rn(cs), ts),
                                       __ddiv_rn(__ull2double_rn(incl[uint64_t(iq) * F + f]), tr));
            w = d > lim;
        }
        want[f] = w;
    }
}
__global__ void k_pair_segflags(uint64_t np, const uint64_t* keys, int LB, uint32_t* flag) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < np; i += uint64_t(gridDim.x) * blockDim.x)
        flag[i] = i == 0 || (keys[i] >> LB) != (keys[i - 1] >> LB);
}
// One warp per (side, name): the reference's running sum, in line order, of
// the precomputed per-line quotients (folded.cpp:48-52).  Lane 0 runs the
// strictly sequential add chain over a 256-value chunk in shared memory while
// all lanes' loads of the next chunk are in flight (issued before the chain,
// stored after it), so the chain never waits on L2.
constexpr int kSegChunk = 256;
constexpr int kSegWarps = 8;
__global__ void __launch_bounds__(kSegWarps * 32) k_pair_segsum(uint64_t nseg, const uint32_t* seg, uint64_t np,
                                                                const uint64_t* keys, int LB, int NB,
                                                                const double* vals,
                                                                uint32_t* out_side_f, double* out_v) {
    __shared__ double buf[kSegWarps][2][kSegChunk];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t g = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; g < nseg; g += nw) {
        const uint64_t a = seg[g], b = g + 1 < nseg ? seg[g + 1] : np;
        double acc = 0.0;
        if (b - a <= 32) {  // short: lane 0 adds the (already loaded) values of the warp
            const double v = a + lane < b ? __ldg(vals + a + lane) : 0.0;
            double vv[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) vv[k] = __shfl_sync(0xffffffffu, v, k);
            const int n = int(b - a);
            for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, vv[k]);
        } else {
#pragma unroll
            for (int j = 0; j < kSegChunk / 32; ++j) {
                const uint64_t x = a + lane + 32 * j;
                buf[w][0][lane + 32 * j] = x < b ? __ldg(vals + x) : 0.0;
            }
            __syncwarp();
            int cur = 0;
            for (uint64_t c = a; c < b; c += kSegChunk) {
                double r[kSegChunk / 32];
#pragma unroll
                for (int j = 0; j < kSegChunk / 32; ++j) {
                    const uint64_t x = c + kSegChunk + lane + 32 * j;
                    r[j] = x < b ? __ldg(vals + x) : 0.0;
                }
                if (lane == 0) {
                    const int n = int(b - c < kSegChunk ? b - c : kSegChunk);
                    const double* q = buf[w][cur];
                    int t = 0;
                    for (; t + 8 <= n; t += 8) {
                        double y[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) y[k] = q[t + k];
#pragma unroll
                        for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, y[k]);
                    }
                    for (; t < n; ++t) acc = __dadd_rn(acc, q[t]);
                }
                __syncwarp();
#pragma unroll
                for (int j = 0; j < kSegChunk / 32; ++j) buf[w][cur ^ 1][lane + 32 * j] = r[j];
                __syncwarp();
                cur ^= 1;
            }
        }
        if (lane == 0) {
            const uint64_t k = keys[a] >> LB;  // side << NB | name
            out_side_f[g] = uint32_t((k >> NB) << 31 | (k & ((1ull << NB) - 1)));
            out_v[g] = acc;
        }
    }
}

// Distributed waterline: per-name partial sums of the local ranks, scattered to
// global name keys (then all-reduced across contexts).
__global__ void k_wl_pass1(uint64_t F, const uint32_t* rows, int R, const unsigned long long* incl,
                           const uint64_t* totals, const uint32_t* gkey, double* s1, unsigned* np) {
    const int lane = threadIdx.x & 31;
    for (uint64_t f = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; f < F;
         f += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        double acc = 0.0;
        unsigned n = 0;
        for (int i0 = 0; i0 < R; i0 += 32) {
            const int i = i0 + lane;
            double x = 0.0;
            bool pres = false;
            if (i < R) {
                const uint32_t r = rows[i];
                const unsigned long long c = incl[uint64_t(r) * F + f];
                pres = c != 0;
                if (pres) x = __ddiv_rn(double(c), double(totals[r]));
            }
            const unsigned m = __ballot_sync(0xffffffffu, pres);
            n += __popc(m);
            acc = warp_ordered_sum(acc, x, m);
        }
        if (lane == 0) {
            s1[gkey[f]] = acc;
            np[gkey[f]] = n;
        }
    }
}
__global__ void k_wl_pass2(uint64_t F, const uint32_t* rows, int R, const unsigned long long* incl,
                           const uint64_t* totals, const uint32_t* gkey, const double* s1, const unsigned* np,
                           double rt, double* s2) {
    const int lane = threadIdx.x & 31;
    for (uint64_t f = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; f < F;
         f += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const uint32_t g = gkey[f];
        const double mu = __ddiv_rn(s1[g], rt);
        double acc = 0.0;
        for (int i0 = 0; i0 < R; i0 += 32) {
            const int i = i0 + lane;
            double dd = 0.0;
            bool pres = false;
            if (i < R) {
                const uint32_t r = rows[i];
                const unsigned long long c = incl[uint64_t(r) * F + f];
                pres = c != 0;
                if (pres) {
                    const double d = __dsub_rn(__ddiv_rn(double(c), double(totals[r])), mu);
                    dd = __dmul_rn(d, d);
                }
            }
            acc = warp_ordered_sum(acc, dd, __ballot_sync(0xffffffffu, pres));
        }
        if (lane == 0) s2[g] = acc;
    }
}
__global__ void k_wl_final(uint64_t NG, const double* s1, const unsigned* np, const double* s2, double rt,
                           double* mean, double* sd) {
    for (uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; g < NG; g += uint64_t(gridDim.x) * blockDim.x) {
        if (!np[g]) {  // name absent everywhere: no waterline entry
            mean[g] = 0.0;
            sd[g] = 0.0;
            continue;
        }
        const double mu = __ddiv_rn(s1[g], rt);
        double v = s2[g];
        for (double k = np[g]; k < rt; k += 1.0) v = __dadd_rn(v, __dmul_rn(mu, mu));
        mean[g] = mu;
        sd[g] = __dsqrt_rn(__ddiv_rn(v, rt));
    }
}
__global__ void k_flag_g(uint64_t F, const uint32_t* rows, int R, const unsigned long long* incl,
                         const uint64_t* totals, double k, const uint32_t* gkey, const double* mean, const double* sd,
                         uint32_t* o_r, uint32_t* o_f, double* o_frac, double* o_thr, unsigned long long* n_out,
                         unsigned long long cap) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < F * uint64_t(R);
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = rows[i / F], f = i % F;
        const unsigned long long c = incl[r * F + f];
        if (!c) continue;
        const uint32_t g = gkey[f];
        const double fr = __ddiv_rn(double(c), double(totals[r]));
        const double thr = __dadd_rn(mean[g], __dmul_rn(k, sd[g]));
        if (fr > thr) {
            const unsigned long long o = atomicAdd(n_out, 1ull);
            if (o < cap) {
                o_r[o] = uint32_t(r);
                o_f[o] = uint32_t(f);
                o_frac[o] = fr;
                o_thr[o] = thr;
            }
        }
    }
}

// Runner::to_global on the device: a local label maps through its global key,
// a dictionary name i to i + (global labels whose dictionary position <= i)
__global__ void k_to_global(uint64_t F, const uint32_t* dense_final, const uint64_t* loc_final,
                            const uint32_t* loc_global, uint64_t nl, const uint32_t* pos, uint64_t ng, uint32_t* out) {
    for (uint64_t f = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; f < F; f += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t fin = dense_final[f];
        uint64_t lo = 0, hi = nl;  // lower_bound(loc_final, fin)
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (loc_final[mid] < fin) lo = mid + 1; else hi = mid;
        }
        if (lo < nl && loc_final[lo] == fin) {
            out[f] = loc_global[lo];
            continue;
        }
        const uint64_t i = fin - lo;
        uint64_t a = 0, b = ng;  // upper_bound(pos, i)
        while (a < b) {
            const uint64_t mid = (a + b) >> 1;
            if (pos[mid] <= i) a = mid + 1; else b = mid;
        }
        out[f] = uint32_t(i + a);
    }
}
__global__ void k_mark_u8(uint64_t n, const uint32_t* idx, uint8_t* map) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        map[idx[i]] = 1;
}
__global__ void k_u8_to_u32(uint64_t n, const uint8_t* a, uint32_t* b) {  // b[n] = 0
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i <= n; i += uint64_t(gridDim.x) * blockDim.x)
        b[i] = i < n ? a[i] : 0u;
}
__global__ void k_scatter_add(uint64_t n, const uint32_t* to, const unsigned long long* v, unsigned long long* out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        atomicAdd(out + to[i], v[i]);
}
__global__ void k_gather_u32(uint64_t n, const uint32_t* idx, const uint32_t* src, uint32_t* out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = src[idx[i]];
}
__global__ void k_u32_to_u64(uint64_t n, const uint32_t* a, unsigned long long* b) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        b[i] = a[i];
}
__global__ void k_clk_of_cpu(int R, const int32_t* rank_ids, const int64_t* off, int64_t* clk) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) clk[r] = off[rank_ids[r]];
}

}  // namespace

void launch_build_buckets(const ulonglong2* e, uint32_t n, uint64_t base, uint32_t shift, uint32_t nb,
                          uint32_t* bucket, cudaStream_t s) {
    k_build_buckets<<<grid_for(uint64_t(nb) + 1), kThreads, 0, s>>>(e, n, base, shift, nb, bucket);
    STG_CUDA(cudaGetLastError());
}

}  // namespace stg

#include "stg_runner.inl"
#include "stg_output.inl"
