// stream_bench.cu -- how fast can one CTA per SM stream HBM into shared memory
// with 1-D bulk async copies (the K5 producer pattern)?  Sweeps ring depth and
// copy size; each CTA consumes (waits on) stages in order and immediately
// re-issues them.  Reports achieved GB/s over a 2 GiB read.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stream_bench tools/stream_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2411_15707_b200/csrc/common.cuh"

using namespace nimbus;

__global__ void __launch_bounds__(128, 1) k_stream(const uint8_t* src, size_t chunk_per_cta, uint32_t stages,
                                                  uint32_t bytes, unsigned long long* sink, int shared = 0) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bars[16];
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < stages; s++) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint8_t* base = shared ? src + (size_t)(blockIdx.x % 4) * 65536 : src + (size_t)blockIdx.x * chunk_per_cta;
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
                                                 uint32_t bytes, unsigned long long* sink, int contiguous = 0) {
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
    const uint32_t tpc = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint32_t t_begin = contiguous ? blockIdx.x * tpc : blockIdx.x;
    const uint32_t t_step = contiguous ? 1 : gridDim.x;
    const uint32_t t_end = contiguous ? min(ntiles, t_begin + tpc) : ntiles;
    for (uint32_t t = t_begin; t < t_end; t += t_step) n += per;
    unsigned long long acc = 0;
    uint32_t t = t_begin, q = 0;
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
            if (++q == per) { q = 0; t += t_step; }
        }
    }
    sink[blockIdx.x] = acc;
}

// touch one 32-byte sector per 64 KB of a region (TLB / page warm-up, negligible bytes)
__global__ void k_touch(const uint8_t* src, size_t bytes, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (size_t off = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 65536; off < bytes;
         off += (size_t)gridDim.x * blockDim.x * 65536)
        acc += src[off];
    if (acc == 12345) sink[0] = acc;
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
    // L2-resident source: every CTA streams the same 8 MB region (L2 hits after the first pass)
    for (uint32_t bytes : {16384u, 32768u, 65536u}) {
        for (uint32_t stages : {2u, 3u, 4u, 6u}) {
            const size_t smem = (size_t)stages * bytes + 1024;
            if (smem > 232448) continue;
            cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            // each CTA: 64 MB total traffic, re-reading an 8 MB window
            const size_t chunk_l2 = (size_t)8 << 20;
            k_stream<<<sms, 128, smem>>>(src, chunk_l2, stages, bytes, sink, 1);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            for (int rep = 0; rep < 8; rep++) k_stream<<<sms, 128, smem>>>(src, chunk_l2, stages, bytes, sink, 1);
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double per_sm = 8.0 * chunk_l2 / (ms * 1e-3);
            printf("L2 %6u B x %u stages: %6.1f GB/s per SM, %7.0f GB/s total\n", bytes, stages, per_sm / 1e9,
                   per_sm * sms / 1e9);
        }
    }
    // short, cold (L2 flushed by a 512 MB read) runs over an Enc(W)-sized buffer
    uint8_t* fl;
    cudaMalloc(&fl, (size_t)512 << 20);
    for (uint32_t mb : {50u, 200u}) {
        const uint32_t tile = 96 * 1024, ntiles = (uint32_t)(((size_t)mb << 20) / tile);
        for (uint32_t variant : {0u, 1u, 2u, 3u}) {
            const int contiguous = variant & 1;
            const uint32_t bytes = (variant & 2) ? 32768 : 16384;
            const uint32_t stages = (variant & 2) ? 4 : 6;
            const size_t smem = (size_t)stages * bytes + 1024;
            cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            float best = 1e9;
            for (int rep = 0; rep < 5; rep++) {
                cudaMemset(fl, rep, (size_t)512 << 20);
                k_stream<<<sms, 128, 65 * 1024>>>(fl, ((size_t)512 << 20) / sms & ~size_t(65535), 4, 16384, sink);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                if (getenv("TOUCH")) { k_touch<<<sms, 128>>>(src, (size_t)ntiles * tile, sink); cudaEventRecord(e0); }
                k_tiles<<<sms, 128, smem>>>(src, ntiles, tile, stages, bytes, sink, contiguous);
                cudaEventRecord(e1);
                cudaDeviceSynchronize();
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("tiles %4u MB, %s, %5u B x %2u stages: %8.2f us  %7.0f GB/s  %s\n", mb,
                   contiguous ? "contiguous" : "strided   ", bytes, stages, best * 1e3,
                   (double)ntiles * tile / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
