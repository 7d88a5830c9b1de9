// kernels.cuh — device building blocks shared by the window pipeline kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "stg_internal.h"

namespace stg {

// splitmix64 finalizer / murmur3 fmix64: two independent 64-bit mixers for the
// 128-bit stack fingerprint.
__device__ __forceinline__ uint64_t mix_a(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t mix_b(uint64_t z) {
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ull;
    return z ^ (z >> 33);
}
// Position-tagged terms of a root-first key sequence.  The fingerprint of a
// sequence is (mix(Σ ta + len), mix(Σ tb + len)): order-sensitive because each
// term carries its position, and two independent 64-bit halves.  salt keys the
// terms (a verification retry re-keys every fingerprint; 0 by default).
__device__ __forceinline__ uint64_t term_a(uint32_t key, uint32_t pos, uint64_t salt = 0) {
    return mix_a(((uint64_t(pos) << 32) | key) ^ 0x9e3779b97f4a7c15ull ^ salt);
}
__device__ __forceinline__ uint64_t term_b(uint32_t key, uint32_t pos, uint64_t salt = 0) {
    return mix_b((((uint64_t(key) << 32) | pos) ^ salt) * 0xd6e8feb86659fd93ull + 0x632be59bd9b4e019ull);
}
__device__ __forceinline__ void fp_finish(uint64_t ha, uint64_t hb, uint64_t len, uint64_t& fa,
                                          uint64_t& fb) {
    fa = mix_a(ha ^ (len * 0xa24baed4963ee407ull));
    fb = mix_b(hb + len * 0x9fb21c651e98df25ull);
    if (fa == 0) fa = 1;
    if (fb == 0) fb = 1;
}

struct UnkSet {
    UnkSlot* slots;
    uint32_t mask;
    uint32_t limit;
    unsigned int* used;
    int* overflow;
};

// Insert-or-get of an unresolved (bin, pc) frame; returns its slot index.
__device__ __forceinline__ uint32_t unk_get(const UnkSet& u, uint32_t bin, uint64_t pc) {
    uint32_t i = uint32_t(mix_a(pc ^ (uint64_t(bin) << 52) ^ 0x5bd1e9955bd1e995ull)) & u.mask;
    for (uint32_t probe = 0; probe <= u.mask; ++probe) {
        volatile UnkSlot* s = u.slots + i;
        uint32_t b = s->bin1;
        if (b == 0) {
            uint32_t prev = atomicCAS(&u.slots[i].bin1, 0u, 0xffffffffu);
            if (prev == 0) {
                s->pc = pc;
                __threadfence();
                atomicExch(&u.slots[i].bin1, bin + 1);
                if (atomicAdd(u.used, 1u) + 1 > u.limit) *u.overflow = 1;
                return i;
            }
            b = prev;
        }
        while (b == 0xffffffffu) {
            __nanosleep(32);
            b = s->bin1;
        }
        __threadfence();
        if (b == bin + 1 && s->pc == pc) return i;
        i = (i + 1) & u.mask;
    }
    *u.overflow = 1;
    return 0;
}

// SymbolFile::lookup (symfile.cpp:54-75) on a staged table: greatest entry with
// start <= pc, then the exact-range / nearest-lower check.  Returns the name
// rank, or kUnknownBit when the frame does not resolve.
__device__ __forceinline__ uint32_t table_lookup(const DevTable& t, uint64_t pc, int mode) {
    if (!t.valid || pc < t.base) return kUnknownBit;  // below first entry (lo == 0)
    uint32_t i;
    uint64_t b = (pc - t.base) >> t.shift;
    if (b >= t.nb) {
        i = t.n - 1;
    } else {
        uint32_t lo = __ldg(t.bucket + b), hi = __ldg(t.bucket + b + 1);
        while (lo < hi) {
            uint32_t mid = (lo + hi + 1) >> 1;
            if (__ldg(&t.e[mid].x) <= pc)
                lo = mid;
            else
                hi = mid - 1;
        }
        i = lo;
    }
    ulonglong2 e = __ldg(t.e + i);
    if (mode == STG_LOOKUP_NEAREST_LOWER) return uint32_t(e.y >> 32);
    uint32_t size = uint32_t(e.y);
    bool in = size == 0 ? pc == e.x : pc < e.x + uint64_t(size);
    return in ? uint32_t(e.y >> 32) : kUnknownBit;
}

// Frame key: name rank, or kUnknownBit | unknown-set slot.
__device__ __forceinline__ uint32_t resolve_frame(const DevTable* tabs, uint32_t n_bins, uint64_t pc,
                                                  uint32_t bin, int mode, const UnkSet& u,
                                                  int* err_bin) {
    uint32_t k = kUnknownBit;
    if (bin < n_bins)
        k = table_lookup(tabs[bin], pc, mode);
    else
        *err_bin = 1;
    if (k == kUnknownBit) k = kUnknownBit | unk_get(u, bin, pc);
    return k;
}

}  // namespace stg
