// membench.cu — ceiling of the HBM access patterns k_sym_agg can use (tools only,
// not product).  Reads a buffer >> L2 with:
//   0  coalesced: a warp reads 1 KB contiguous per 256-bit load instruction
//   1  lane-strided: lane s reads its own 512 B record, 32 B per instruction
//      (k_sym_agg's frame loads)
//   2  bulk copy: each warp stages its 16 KB block into shared memory with
//      cp.async.bulk (double buffered, mbarrier completion), lanes read smem
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/membench.cu -o /tmp/membench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

// blocks of 32 records x 512 B = 16 KB per warp iteration
__global__ void k_coalesced(const uint64_t* buf, uint64_t n_blocks, uint64_t* out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    uint64_t acc = 0;
    for (uint64_t b = warp; b < n_blocks; b += nw) {
        const uint64_t* base = buf + b * 2048;
#pragma unroll 4
        for (int k = 0; k < 16; ++k) {
            uint64_t x, y, z, w;
            ld256(base + k * 128 + lane * 4, x, y, z, w);
            acc ^= x + y * 3 + z * 5 + w * 7;
        }
    }
    if (acc == 0x12345) out[0] = acc;
}

__global__ void k_strided(const uint64_t* buf, uint64_t n_blocks, uint64_t* out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    uint64_t acc = 0;
    for (uint64_t b = warp; b < n_blocks; b += nw) {
        const uint64_t* base = buf + b * 2048 + lane * 64;
#pragma unroll 4
        for (int k = 0; k < 16; ++k) {
            uint64_t x, y, z, w;
            ld256(base + k * 4, x, y, z, w);
            acc ^= x + y * 3 + z * 5 + w * 7;
        }
    }
    if (acc == 0x12345) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(bar)),
        "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}

template <int WPB, int STAGES, int CHUNK>
__global__ void k_bulk(const uint64_t* buf, uint64_t n_blocks, uint64_t* out) {
    // CHUNK bytes per stage per warp
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[WPB][STAGES];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char* my = smem + size_t(wid) * STAGES * CHUNK;
    if (lane == 0)
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[wid][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint64_t warp = blockIdx.x * uint64_t(WPB) + wid;
    const uint64_t nw = uint64_t(gridDim.x) * WPB;
    const uint64_t total = n_blocks * 16384ull / CHUNK;  // chunks
    uint64_t acc = 0;
    // prologue
    uint64_t c = warp;
    for (int s = 0; s < STAGES; ++s) {
        uint64_t cc = c + uint64_t(s) * nw;
        if (lane == 0 && cc < total) {
            mbar_expect_tx(&bars[wid][s], CHUNK);
            bulk_g2s(my + s * CHUNK, reinterpret_cast<const unsigned char*>(buf) + cc * CHUNK, CHUNK, &bars[wid][s]);
        }
    }
    unsigned phase = 0;
    int s = 0;
    for (; c < total; c += nw) {
        mbar_wait(&bars[wid][s], phase);
        const uint4* q = reinterpret_cast<const uint4*>(my + s * CHUNK);
#pragma unroll 4
        for (int k = lane; k < CHUNK / 16; k += 32) {
            uint4 v = q[k];
            acc ^= v.x + v.y * 3ull + v.z * 5ull + v.w * 7ull;
        }
        __syncwarp();
        uint64_t nx = c + uint64_t(STAGES) * nw;
        if (lane == 0 && nx < total) {
            mbar_expect_tx(&bars[wid][s], CHUNK);
            bulk_g2s(my + s * CHUNK, reinterpret_cast<const unsigned char*>(buf) + nx * CHUNK, CHUNK, &bars[wid][s]);
        }
        if (++s == STAGES) {
            s = 0;
            phase ^= 1;
        }
    }
    if (acc == 0x12345) out[0] = acc;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    const uint64_t bytes = 16ull << 30;
    uint64_t* buf;
    uint64_t* out;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&out, 64);
    cudaMemset(buf, 1, bytes);
    const uint64_t nb = bytes / 16384;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cta : {4, 8, 16}) {
        float ms = timeit([&] { k_coalesced<<<sms * cta, 256>>>(buf, nb, out); });
        printf("coalesced   grid %3d x 256: %.3f ms  %.0f GB/s\n", cta, ms, bytes / ms / 1e6);
        ms = timeit([&] { k_strided<<<sms * cta, 256>>>(buf, nb, out); });
        printf("lane-stride grid %3d x 256: %.3f ms  %.0f GB/s\n", cta, ms, bytes / ms / 1e6);
    }
    {
        constexpr int WPB = 8, ST = 2, CH = 8192;
        size_t sm = size_t(WPB) * ST * CH;
        cudaFuncSetAttribute(k_bulk<WPB, ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        for (int cta : {1, 2}) {
            float ms = timeit([&] { k_bulk<WPB, ST, CH><<<sms * cta, WPB * 32, sm>>>(buf, nb, out); });
            printf("bulk 8w x 2st x 8KB, %d CTA/SM: %.3f ms  %.0f GB/s (%s)\n", cta, ms, bytes / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    {
        constexpr int WPB = 8, ST = 3, CH = 4096;
        size_t sm = size_t(WPB) * ST * CH;
        cudaFuncSetAttribute(k_bulk<WPB, ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        for (int cta : {1, 2}) {
            float ms = timeit([&] { k_bulk<WPB, ST, CH><<<sms * cta, WPB * 32, sm>>>(buf, nb, out); });
            printf("bulk 8w x 3st x 4KB, %d CTA/SM: %.3f ms  %.0f GB/s (%s)\n", cta, ms, bytes / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    {
        constexpr int WPB = 4, ST = 4, CH = 8192;
        size_t sm = size_t(WPB) * ST * CH;
        cudaFuncSetAttribute(k_bulk<WPB, ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        for (int cta : {1, 2}) {
            float ms = timeit([&] { k_bulk<WPB, ST, CH><<<sms * cta, WPB * 32, sm>>>(buf, nb, out); });
            printf("bulk 4w x 4st x 8KB, %d CTA/SM: %.3f ms  %.0f GB/s (%s)\n", cta, ms, bytes / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
