// stream_bench.cu -- how fast can one CTA per SM stream HBM into shared memory
// with 1-D bulk async copies (the K5 producer pattern)?  Sweeps ring depth and
// copy size; each CTA consumes (waits on) stages in order and immediately
// re-issues them.  Reports achieved GB/s over a 2 GiB read.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stream_bench tools/stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2411_15707_b200/csrc/common.cuh"

using namespace nimbus;

__global__ void __launch_bounds__(128, 1) k_stream(const uint8_t* src, size_t chunk_per_cta, uint32_t stages,
                                                  uint32_t bytes, unsigned long long* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bars[16];
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < stages; s++) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint8_t* base = src + (size_t)blockIdx.x * chunk_per_cta;
    const uint32_t n = (uint32_t)(chunk_per_cta / bytes);
    const uint64_t pol = policy_evict_first();
    unsigned long long acc = 0;
    for (uint32_t i = 0; i < n + stages; i++) {
        if (i >= stages) {
            const uint32_t j = i - stages, s = j % stages;
            mbar_wait(&bars[s], (j / stages) & 1);
            acc += smem[s * bytes];
        }
        if (i < n) {
            const uint32_t s = i % stages;
            mbar_arrive_expect_tx(&bars[s], bytes);
            bulk_g2s(smem + s * bytes, base + (size_t)i * bytes, bytes, &bars[s], pol);
        }
    }
    sink[blockIdx.x] = acc;
}

// Enc(W)-like pattern: CTA c streams tiles c, c + grid, ... of `tile` bytes each.
__global__ void __launch_bounds__(128, 1) k_tiles(const uint8_t* src, uint32_t ntiles, uint32_t tile, uint32_t stages,
                                                 uint32_t bytes, unsigned long long* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bars[16];
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < stages; s++) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint64_t pol = policy_evict_first();
    const uint32_t per = tile / bytes;
    uint32_t n = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) n += per;
    unsigned long long acc = 0;
    uint32_t t = blockIdx.x, q = 0;
    for (uint32_t i = 0; i < n + stages; i++) {
        if (i >= stages) {
            const uint32_t j = i - stages, s = j % stages;
            mbar_wait(&bars[s], (j / stages) & 1);
            acc += smem[s * bytes];
        }
        if (i < n) {
            const uint32_t s = i % stages;
            mbar_arrive_expect_tx(&bars[s], bytes);
            bulk_g2s(smem + s * bytes, src + (size_t)t * tile + (size_t)q * bytes, bytes, &bars[s], pol);
            if (++q == per) { q = 0; t += gridDim.x; }
        }
    }
    sink[blockIdx.x] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t total = (size_t)2 << 30;
    uint8_t* src;
    cudaMalloc(&src, total);
    cudaMemset(src, 1, total);
    unsigned long long* sink;
    cudaMalloc(&sink, 8 * 1024);
    const size_t chunk = (total / sms) & ~size_t(65535);
    for (uint32_t bytes : {8192u, 16384u, 32768u, 65536u}) {
        for (uint32_t stages : {2u, 3u, 4u, 6u, 8u, 12u}) {
            const size_t smem = (size_t)stages * bytes + 1024;
            if (smem > 232448 || stages > 16) continue;
            cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_stream<<<sms, 128, smem>>>(src, chunk, stages, bytes, sink);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_stream<<<sms, 128, smem>>>(src, chunk, stages, bytes, sink);
            cudaEventRecord(e1);
            cudaError_t err = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("copy %6u B x %2u stages (%4u KB in flight/SM): %7.0f GB/s  %s\n", bytes, stages,
                   stages * bytes / 1024, (double)chunk * sms / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
        }
    }
    // short, cold (L2 flushed by a 512 MB read) runs over an Enc(W)-sized buffer
    uint8_t* fl;
    cudaMalloc(&fl, (size_t)512 << 20);
    for (uint32_t mb : {50u, 200u, 600u}) {
        const uint32_t tile = 96 * 1024, ntiles = (uint32_t)(((size_t)mb << 20) / tile);
        for (uint32_t stages : {5u, 8u, 12u}) {
            const uint32_t bytes = 16384;
            const size_t smem = (size_t)stages * bytes + 1024;
            cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            float best = 1e9;
            for (int rep = 0; rep < 5; rep++) {
                cudaMemset(fl, rep, (size_t)512 << 20);
                k_stream<<<sms, 128, 65 * 1024>>>(fl, ((size_t)512 << 20) / sms & ~size_t(65535), 4, 16384, sink);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                k_tiles<<<sms, 128, smem>>>(src, ntiles, tile, stages, bytes, sink);
                cudaEventRecord(e1);
                cudaDeviceSynchronize();
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("tiles %4u MB, 96 KB tiles, 16 KB x %2u stages: %8.2f us  %7.0f GB/s  %s\n", mb, stages, best * 1e3,
                   (double)ntiles * tile / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
