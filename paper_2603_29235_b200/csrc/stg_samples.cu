// stg_samples.cu — the raw-address ProfileWindow API:
//
//   std::vector<ProfileWindow> aggregate_samples(stream, drain_interval_ns)
//                                              samples.hpp:38-44, samples.cpp:31-85
//
// One rank's time-ordered stream of raw stacks (FrameRef = (build id, offset),
// vprocess.hpp:48-53) is cut on the drain grid and, per window, identical stacks
// merge into one record; records keep FIRST-SEEN order and the counts sum to the
// number of input samples (lossless: the reference falls back to full-stack
// comparison on digest collisions, samples.cpp:69-76).
//
// Device algorithm (HBM-bound: ~10 B per frame + 16 B per sample read once; the
// verification re-reads a sample's frames from L1 and its representative's from L2):
//   1. k_agg_hash — lane per sample: validation in the reference's order (empty
//      stack, mixed ranks, timestamp regression; the first bad sample in stream
//      order wins), window index on the drain grid, 128-bit position-tagged
//      fingerprint of (window, (bin, offset)...), warp pre-aggregation of equal
//      fingerprints (__match_any) and one insert per group into an open-addressing
//      table whose slot keeps the minimum sample index (first seen) and the count.
//   2. in the same kernel, every sample compares its frames with a representative
//      of its slot; any difference (a 128-bit collision) switches the call to the
//      exact path below, so the result never depends on the fingerprint.
//   3. k_agg_flags + scan + k_agg_records — a sample that is its slot's first is a
//      record; sample order = (window, first-seen) order, i.e. the reference's.
//   4. window heads over the records -> window starts/ends and record offsets.
// Exact path (collisions, or forced for tests): merge sort of sample indices by
// (window, frames) with a full comparator; equal runs are records (stable sort:
// the run head is the first-seen sample).
#include <cub/cub.cuh>

#include <algorithm>
#include <string>

#include "kernels.cuh"
#include "stg_internal.h"

namespace stg {
namespace {

constexpr int kT = 256;
inline unsigned grid_of(uint64_t n, int per = kT) {
    uint64_t g = (n + per - 1) / per;
    return unsigned(g < 1 ? 1 : (g > 148ull * 64 ? 148ull * 64 : g));
}

// Zero-initialised slot.  The 16-byte key is claimed or read by ONE 128-bit
// CAS, so no ready flag and no fences; the first-seen index is kept inverted
// (atomicMax of ~i == min i) so that zero means "none yet".
struct __align__(32) RawSlot {
    unsigned long long ka, kb;       // fingerprint; (0, 0) = empty
    unsigned long long first_inv;    // ~(min sample index)
    unsigned int count;
    unsigned int pad;
};

// atom.global.cas.b128: returns the previous key
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

struct Stream {
    const int64_t* ts;
    const int32_t* rank;
    const uint64_t* foff;
    const uint64_t* pc;
    const uint16_t* bin;
    uint64_t n;
    uint64_t n_frames;
    int64_t w0;      // start of the first window (floor-aligned first timestamp)
    int64_t drain;
};

__device__ __forceinline__ uint64_t win_of(const Stream& s, uint64_t i) {
    return uint64_t((s.ts[i] - s.w0) / s.drain);
}

// One 64-bit mix per frame; the fingerprint is (Σ t, Σ rotr(t, 29)).  Its
// quality only matters for speed: every sample is verified frame by frame.
// (pos wraps at 2^16 frames per stack; the verification covers that too.)
__device__ __forceinline__ uint64_t raw_term(uint64_t pc, uint32_t bin, uint32_t pos) {
    return mix_a(pc ^ (uint64_t(bin | (pos << 16)) << 32) ^ 0x3c6ef372fe94f82bull);
}
__device__ __forceinline__ void raw_add(uint64_t& ha, uint64_t& hb, uint64_t t) {
    ha += t;
    hb += (t >> 29) | (t << 35);
}

// 256-bit read-only global load (LDG.E.ENL2.256), 32-byte aligned address;
// L1-allocating, so the verification pass re-reads the sample from L1.
__device__ __forceinline__ void ld256(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d) {
    asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
}

constexpr int kAggWarps = kT / 32;

// Warp w owns a contiguous range of 32-sample batches, so concurrent warps work
// in different windows and their slot atomics spread over many slots (a
// grid-stride order puts every warp in the same window, on the same few slots).
// Lane = sample:
//   phase 1  validation, window, fingerprint over the sample's frames;
//   phase 2  warp grouping of equal fingerprints, one table insert per group;
//   phase 3  the sample's frames (now in L1) against the slot's representative
//            (L2): any difference flags a collision.
template <bool ALIGNED>
__global__ void __launch_bounds__(kT) k_agg_hash(Stream s, RawSlot* T, uint64_t mask, uint32_t* slot_of,
                                                 unsigned long long* err, int* overflow, int* mismatch,
                                                 unsigned* used, unsigned limit) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t n_batches = (s.n + 31) / 32;
    const uint64_t per = (n_batches + nw - 1) / nw;
    const uint64_t b0 = warp * per, b1 = min(n_batches, b0 + per);
    for (uint64_t b = b0; b < b1; ++b) {
        const uint64_t i = b * 32 + lane;
        const bool live = i < s.n;
        uint64_t fa = 0, fb = 0, w = 0, f0 = 0, f1 = 0;
        // ---- phase 1
        if (live) {
            f0 = __ldg(s.foff + i);
            f1 = __ldg(s.foff + i + 1);
            const bool bad = f1 == f0 || (s.rank && s.rank[i] != s.rank[0]) || (i > 0 && s.ts[i] < s.ts[i - 1]);
            if (bad) atomicMin(err, (unsigned long long)i);
            w = win_of(s, i);
            uint64_t ha = mix_a(w ^ 0x5851f42d4c957f2dull), hb = mix_b(w + 0x14057b7ef767814full);
            if (ALIGNED) {
                // blocks of 8 frames: two 256-bit pc loads + one 16-byte bin load per
                // lane, each a whole sector (the frames of one lane are contiguous)
                for (uint64_t blk = f0 & ~7ull; blk < f1; blk += 8) {
                    uint64_t pcs[8];
                    uint32_t bns[8];
                    if (blk + 8 <= s.n_frames) {
                        ld256(s.pc + blk, pcs[0], pcs[1], pcs[2], pcs[3]);
                        ld256(s.pc + blk + 4, pcs[4], pcs[5], pcs[6], pcs[7]);
                        const uint4 bq = __ldg(reinterpret_cast<const uint4*>(s.bin + blk));
                        bns[0] = bq.x & 0xffffu; bns[1] = bq.x >> 16; bns[2] = bq.y & 0xffffu; bns[3] = bq.y >> 16;
                        bns[4] = bq.z & 0xffffu; bns[5] = bq.z >> 16; bns[6] = bq.w & 0xffffu; bns[7] = bq.w >> 16;
                    } else {
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            pcs[t] = blk + t < s.n_frames ? s.pc[blk + t] : 0;
                            bns[t] = blk + t < s.n_frames ? s.bin[blk + t] : 0;
                        }
                    }
                    const uint32_t pos0 = uint32_t(blk - f0);
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        const uint64_t m = (blk + t >= f0 && blk + t < f1) ? ~0ull : 0ull;
                        raw_add(ha, hb, raw_term(pcs[t], bns[t], pos0 + t) & m);
                    }
                }
            } else {
                for (uint64_t f = f0; f < f1; ++f)
                    raw_add(ha, hb, raw_term(__ldg(s.pc + f), __ldg(s.bin + f), uint32_t(f - f0)));
            }
            fp_finish(ha, hb, f1 - f0, fa, fb);
        }
        // ---- phase 2
        const unsigned act = __ballot_sync(0xffffffffu, live);
        const unsigned grp = __match_any_sync(0xffffffffu, live ? fa : 0ull) &
                             __match_any_sync(0xffffffffu, live ? fb : 0ull) & act;
        const int leader = live ? __ffs(grp) - 1 : lane;
        uint32_t slot = 0;
        unsigned long long rep = i;
        if (live && leader == lane) {
            uint64_t h = mix_a(fa ^ (fb >> 7)) & mask;
            bool done = false;
            for (uint64_t probe = 0; probe <= mask; ++probe) {
                unsigned long long oa, ob;
                cas128(&T[h].ka, fa, fb, oa, ob);
                if ((oa | ob) == 0) {  // claimed an empty slot
                    if (atomicAdd(used, 1u) + 1 > limit) *overflow = 1;
                }
                if ((oa | ob) == 0 || (oa == fa && ob == fb)) {
                    // any member is a valid representative: if the slot held a
                    // colliding stack, some comparison below differs
                    const unsigned long long prev = atomicMax(&T[h].first_inv, ~(unsigned long long)i);
                    atomicAdd(&T[h].count, unsigned(__popc(grp)));
                    if (prev != 0) rep = ~prev;
                    done = true;
                    break;
                }
                if (*(volatile int*)overflow) break;  // the host retries with a larger table
                h = (h + 1) & mask;
            }
            if (!done) *overflow = 1;
            slot = uint32_t(h);
        }
        slot = __shfl_sync(0xffffffffu, slot, leader);
        rep = __shfl_sync(0xffffffffu, rep, leader);
        // ---- phase 3
        if (live) {
            slot_of[i] = slot;
            if (rep != i) {
                const uint64_t r0 = __ldg(s.foff + rep), r1 = __ldg(s.foff + rep + 1), len = f1 - f0;
                uint64_t diff = (r1 - r0 != len || win_of(s, rep) != w) ? 1 : 0;
                // blocks of 8 frames, all 32 loads in flight (own frames from L1)
                for (uint64_t k = 0; !diff && k < len; k += 8) {
                    uint64_t a[8], b[8];
                    uint32_t x[8], y[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        const bool v = k + t < len;
                        a[t] = v ? __ldg(s.pc + f0 + k + t) : 0;
                        b[t] = v ? __ldg(s.pc + r0 + k + t) : 0;
                        x[t] = v ? __ldg(s.bin + f0 + k + t) : 0;
                        y[t] = v ? __ldg(s.bin + r0 + k + t) : 0;
                    }
#pragma unroll
                    for (int t = 0; t < 8; ++t) diff |= (a[t] ^ b[t]) | uint64_t(x[t] ^ y[t]);
                }
                if (diff) *mismatch = 1;
            }
        }
    }
}

__global__ void k_agg_flags(uint64_t n, const RawSlot* T, const uint32_t* slot_of, uint32_t* flag) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        flag[i] = ~T[slot_of[i]].first_inv == i ? 1u : 0u;
}

__global__ void k_agg_records(Stream s, const RawSlot* T, const uint32_t* slot_of, const uint32_t* flag,
                              const uint32_t* pos, uint64_t* rec_first, uint64_t* rec_count, uint64_t* rec_win) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < s.n; i += uint64_t(gridDim.x) * blockDim.x)
        if (flag[i]) {
            const uint32_t r = pos[i];
            rec_first[r] = i;
            rec_count[r] = T[slot_of[i]].count;
            rec_win[r] = win_of(s, i);
        }
}

__device__ __forceinline__ bool same_stack(const Stream& s, uint64_t a, uint64_t b) {
    const uint64_t a0 = s.foff[a], a1 = s.foff[a + 1], b0 = s.foff[b], b1 = s.foff[b + 1];
    if (a1 - a0 != b1 - b0) return false;
    for (uint64_t k = 0; k < a1 - a0; ++k)
        if (s.pc[a0 + k] != s.pc[b0 + k] || s.bin[a0 + k] != s.bin[b0 + k]) return false;
    return true;
}

// ---- exact path: sort sample indices by (window, frames)
struct StackLess {
    Stream s;
    __device__ bool operator()(uint32_t a, uint32_t b) const {
        const uint64_t wa = win_of(s, a), wb = win_of(s, b);
        if (wa != wb) return wa < wb;
        const uint64_t a0 = s.foff[a], a1 = s.foff[a + 1], b0 = s.foff[b], b1 = s.foff[b + 1];
        const uint64_t la = a1 - a0, lb = b1 - b0, m = la < lb ? la : lb;
        for (uint64_t k = 0; k < m; ++k) {
            const uint16_t xa = s.bin[a0 + k], xb = s.bin[b0 + k];
            if (xa != xb) return xa < xb;
            const uint64_t pa = s.pc[a0 + k], pb = s.pc[b0 + k];
            if (pa != pb) return pa < pb;
        }
        return la < lb;
    }
};

// Run heads of the sorted order become records: the head (smallest index, the
// sort is stable) is marked in flag[], the run length goes to run_count[head].
__global__ void k_exact_runs(Stream s, const uint32_t* sorted, uint32_t* flag, uint32_t* run_count) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < s.n; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t i = sorted[j];
        const bool head = j == 0 || win_of(s, sorted[j - 1]) != win_of(s, i) || !same_stack(s, sorted[j - 1], i);
        if (!head) continue;
        uint64_t e = j + 1;
        while (e < s.n && win_of(s, sorted[e]) == win_of(s, i) && same_stack(s, sorted[e], i)) ++e;
        flag[i] = 1;
        run_count[i] = uint32_t(e - j);
    }
}

__global__ void k_exact_records(Stream s, const uint32_t* flag, const uint32_t* pos, const uint32_t* run_count,
                                uint64_t* rec_first, uint64_t* rec_count, uint64_t* rec_win) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < s.n; i += uint64_t(gridDim.x) * blockDim.x)
        if (flag[i]) {
            const uint32_t r = pos[i];
            rec_first[r] = i;
            rec_count[r] = run_count[i];
            rec_win[r] = win_of(s, i);
        }
}

__global__ void k_win_heads(uint64_t R, const uint64_t* rec_win, uint32_t* head) {
    for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < R; r += uint64_t(gridDim.x) * blockDim.x)
        head[r] = (r == 0 || rec_win[r] != rec_win[r - 1]) ? 1u : 0u;
}

__global__ void k_win_fill(uint64_t R, const uint64_t* rec_win, const uint32_t* head, const uint32_t* widx,
                           int64_t w0, int64_t drain, int64_t* ws, int64_t* we, uint64_t* rec_off) {
    for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < R; r += uint64_t(gridDim.x) * blockDim.x)
        if (head[r]) {
            const uint32_t w = widx[r];
            ws[w] = w0 + int64_t(rec_win[r]) * drain;
            we[w] = ws[w] + drain;
            rec_off[w] = r;
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

void* scratch(Ctx& c, size_t bytes) { return c.buf("ag_tmp").get(bytes ? bytes : 1); }

// Exclusive positions of flag[0, n) (flag has n + 1 cells; the last is zeroed);
// returns the number of set flags.
uint64_t compact_positions(Ctx& c, uint32_t* flag, uint32_t* pos, uint64_t n) {
    STG_CUDA(cudaMemsetAsync(flag + n, 0, 4, c.stream));
    size_t tb = 0;
    STG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, int64_t(n + 1), c.stream));
    STG_CUDA(cub::DeviceScan::ExclusiveSum(scratch(c, tb), tb, flag, pos, int64_t(n + 1), c.stream));
    return get1(c, pos + n);
}

__global__ void k_iota32(uint64_t n, uint32_t* v) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        v[i] = uint32_t(i);
}

template <class T>
const T* to_device(Ctx& c, const char* name, const T* p, uint64_t n, bool host) {
    if (!host || !p) return p;
    T* d = dbuf<T>(c, name, n);
    if (n) STG_CUDA(cudaMemcpyAsync(d, p, n * sizeof(T), cudaMemcpyHostToDevice, c.stream));
    return d;
}

}  // namespace

void aggregate_samples(Ctx& c, const stg_stream& in, int64_t drain, int flags, uint64_t* n_windows,
                       uint64_t* n_records) {
    c.ag_windows = c.ag_records = 0;
    c.ag_valid = false;
    if (drain <= 0) fail(STG_EINVAL, "drain interval must be positive");
    const uint64_t n = in.n_samples;
    if (n >= (1ull << 32)) fail(STG_EINVAL, "aggregate_samples: more than 2^32 - 1 samples per call");
    if (n == 0) {
        c.ag_valid = true;
        *n_windows = *n_records = 0;
        return;
    }
    if (in.memory != STG_MEM_HOST && in.memory != STG_MEM_DEVICE) fail(STG_EINVAL, "unknown stg_stream.memory");
    if (!in.ts || !in.frame_off || !in.frame_pc || !in.frame_bin) fail(STG_EINVAL, "stg_stream: null array");
    const bool host = in.memory == STG_MEM_HOST;
    cudaStream_t st = c.stream;
    // the first window starts at the floor-aligned first timestamp (samples.cpp:37-40)
    int64_t ts0;
    uint64_t nf = 0;
    if (host) {
        ts0 = in.ts[0];
        nf = in.frame_off[n];
    } else {
        STG_CUDA(cudaMemcpyAsync(&ts0, in.ts, 8, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaMemcpyAsync(&nf, in.frame_off + n, 8, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
    }
    Stream s;
    s.n = n;
    s.n_frames = nf;
    s.drain = drain;
    s.w0 = ts0 - ((ts0 % drain + drain) % drain);
    s.ts = to_device(c, "ag_ts", in.ts, n, host);
    s.rank = to_device(c, "ag_rank", in.rank, n, host);
    s.foff = to_device(c, "ag_foff", in.frame_off, n + 1, host);
    s.pc = to_device(c, "ag_pc", in.frame_pc, nf, host);
    s.bin = to_device(c, "ag_bin", in.frame_bin, nf, host);

    unsigned long long* err = dbuf<unsigned long long>(c, "ag_err", 1);
    int* ovf = dbuf<int>(c, "ag_ovf", 4);  // overflow, mismatch, used slots
    uint32_t* slot_of = dbuf<uint32_t>(c, "ag_slot_of", n);
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c.device);
    // the blocked 256-bit loads need frame_pc 32-byte and frame_bin 16-byte aligned
    // (always true for host input, staged into fresh allocations)
    const bool aligned = (reinterpret_cast<uintptr_t>(s.pc) % 32 == 0) && (reinterpret_cast<uintptr_t>(s.bin) % 16 == 0);
    // The table starts at the size the last call needed (clearing 2n slots would
    // cost more than the aggregation for low-cardinality streams) and grows 8x
    // when it passes 3/4 full; 2n slots can never overflow.
    uint64_t cap_max = 1024;
    while (cap_max < 2 * n) cap_max <<= 1;
    uint64_t cap = std::min(cap_max, std::max<uint64_t>(1024, c.ag_cap_hint));
    RawSlot* T;
    int flags2[3];
    for (;;) {
        STG_CUDA(cudaMemsetAsync(err, 0xff, 8, st));
        STG_CUDA(cudaMemsetAsync(ovf, 0, 16, st));
        T = dbuf<RawSlot>(c, "ag_slots", cap);
        STG_CUDA(cudaMemsetAsync(T, 0, cap * sizeof(RawSlot), st));
        const unsigned limit = unsigned(std::min<uint64_t>(cap - cap / 4, 0xffffffffu));
        if (aligned)
            k_agg_hash<true><<<unsigned(dev_sms) * 8, kT, 0, st>>>(s, T, cap - 1, slot_of, err, ovf, ovf + 1,
                                                                   reinterpret_cast<unsigned*>(ovf + 2), limit);
        else
            k_agg_hash<false><<<unsigned(dev_sms) * 8, kT, 0, st>>>(s, T, cap - 1, slot_of, err, ovf, ovf + 1,
                                                                    reinterpret_cast<unsigned*>(ovf + 2), limit);
        STG_CUDA(cudaGetLastError());
        STG_CUDA(cudaMemcpyAsync(flags2, ovf, 12, cudaMemcpyDeviceToHost, st));
        STG_CUDA(cudaStreamSynchronize(st));
        if (!flags2[0] || cap >= cap_max) break;
        cap = std::min(cap_max, cap * 8);
        c.ag_cap_hint = cap;
    }
    STG_CUDA(cudaGetLastError());
    const unsigned long long e = get1(c, err);
    if (e != ~0ull) {
        // the reference's per-sample check order (samples.cpp:55-60)
        uint64_t fo[2];
        int64_t tt[2] = {0, 0};
        int32_t rk[2] = {0, 0};
        STG_CUDA(cudaMemcpyAsync(fo, s.foff + e, 16, cudaMemcpyDeviceToHost, st));
        if (e > 0) STG_CUDA(cudaMemcpyAsync(tt, s.ts + e - 1, 16, cudaMemcpyDeviceToHost, st));
        if (s.rank) {
            STG_CUDA(cudaMemcpyAsync(&rk[0], s.rank, 4, cudaMemcpyDeviceToHost, st));
            STG_CUDA(cudaMemcpyAsync(&rk[1], s.rank + e, 4, cudaMemcpyDeviceToHost, st));
        }
        STG_CUDA(cudaStreamSynchronize(st));
        if (fo[1] == fo[0]) fail(STG_EINVAL, "empty sample stack");
        if (rk[1] != rk[0]) fail(STG_EINVAL, "aggregate_samples: mixed ranks");
        fail(STG_EINVAL, "aggregate_samples: timestamps regressed");
    }
    if (flags2[0]) fail(STG_ENOMEM, "aggregate_samples: hash table overflow");
    const bool exact = (flags & STG_AGG_FORCE_EXACT) || flags2[1] != 0;
    uint32_t* flag = dbuf<uint32_t>(c, "ag_flag", n + 1);
    uint32_t* pos = dbuf<uint32_t>(c, "ag_pos", n + 1);
    uint64_t R;
    uint64_t *rec_first, *rec_count, *rec_win;
    auto records = [&](uint64_t r) {
        rec_first = dbuf<uint64_t>(c, "ag_rec_first", r);
        rec_count = dbuf<uint64_t>(c, "ag_rec_count", r);
        rec_win = dbuf<uint64_t>(c, "ag_rec_win", r);
    };
    if (!exact) {
        k_agg_flags<<<grid_of(n), kT, 0, st>>>(n, T, slot_of, flag);
        R = compact_positions(c, flag, pos, n);
        records(R);
        k_agg_records<<<grid_of(n), kT, 0, st>>>(s, T, slot_of, flag, pos, rec_first, rec_count, rec_win);
    } else {
        uint32_t* idx = dbuf<uint32_t>(c, "ag_idx", n);
        uint32_t* run = dbuf<uint32_t>(c, "ag_run", n);
        k_iota32<<<grid_of(n), kT, 0, st>>>(n, idx);
        size_t tb = 0;
        StackLess less{s};
        STG_CUDA(cub::DeviceMergeSort::StableSortKeys(nullptr, tb, idx, int64_t(n), less, st));
        STG_CUDA(cub::DeviceMergeSort::StableSortKeys(scratch(c, tb), tb, idx, int64_t(n), less, st));
        STG_CUDA(cudaMemsetAsync(flag, 0, n * 4, st));
        k_exact_runs<<<grid_of(n), kT, 0, st>>>(s, idx, flag, run);
        R = compact_positions(c, flag, pos, n);
        records(R);
        k_exact_records<<<grid_of(n), kT, 0, st>>>(s, flag, pos, run, rec_first, rec_count, rec_win);
    }
    STG_CUDA(cudaGetLastError());
    // windows = runs of equal window index over the records (samples.cpp:61-68)
    uint32_t* head = dbuf<uint32_t>(c, "ag_whead", R + 1);
    uint32_t* wx = dbuf<uint32_t>(c, "ag_wx", R + 1);
    k_win_heads<<<grid_of(R), kT, 0, st>>>(R, rec_win, head);
    const uint64_t W = compact_positions(c, head, wx, R);
    int64_t* ws = dbuf<int64_t>(c, "ag_ws", W);
    int64_t* we = dbuf<int64_t>(c, "ag_we", W);
    uint64_t* roff = dbuf<uint64_t>(c, "ag_roff", W + 1);
    k_win_fill<<<grid_of(R), kT, 0, st>>>(R, rec_win, head, wx, s.w0, drain, ws, we, roff);
    STG_CUDA(cudaMemcpyAsync(roff + W, &R, 8, cudaMemcpyHostToDevice, st));
    STG_CUDA(cudaStreamSynchronize(st));
    STG_CUDA(cudaGetLastError());
    c.ag_windows = W;
    c.ag_records = R;
    c.ag_exact = exact;
    c.ag_valid = true;
    *n_windows = W;
    *n_records = R;
}

void aggregate_windows(Ctx& c, int64_t* start, int64_t* end, uint64_t* rec_off) {
    if (!c.ag_valid) fail(STG_ESTATE, "no aggregate_samples result on this context");
    const uint64_t W = c.ag_windows;
    cudaStream_t st = c.stream;
    if (W) {
        if (start) STG_CUDA(cudaMemcpyAsync(start, c.buf("ag_ws").p, W * 8, cudaMemcpyDeviceToHost, st));
        if (end) STG_CUDA(cudaMemcpyAsync(end, c.buf("ag_we").p, W * 8, cudaMemcpyDeviceToHost, st));
        if (rec_off) STG_CUDA(cudaMemcpyAsync(rec_off, c.buf("ag_roff").p, (W + 1) * 8, cudaMemcpyDeviceToHost, st));
    } else if (rec_off) {
        rec_off[0] = 0;
    }
    STG_CUDA(cudaStreamSynchronize(st));
}

void aggregate_records(Ctx& c, uint64_t* first_sample, uint64_t* count) {
    if (!c.ag_valid) fail(STG_ESTATE, "no aggregate_samples result on this context");
    const uint64_t R = c.ag_records;
    cudaStream_t st = c.stream;
    if (R) {
        if (first_sample)
            STG_CUDA(cudaMemcpyAsync(first_sample, c.buf("ag_rec_first").p, R * 8, cudaMemcpyDeviceToHost, st));
        if (count) STG_CUDA(cudaMemcpyAsync(count, c.buf("ag_rec_count").p, R * 8, cudaMemcpyDeviceToHost, st));
    }
    STG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace stg
