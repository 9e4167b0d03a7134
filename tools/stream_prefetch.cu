// stream_prefetch.cu -- can a cold 50 MB stream (the C2/C3 Enc(W) read) beat the
// ~13.2 us bulk-copy floor of tools/stream_cold.cu?  Compares, on the same
// rotated 50 MB copies with a 512 MB read flush before every run:
//   tiles      : 148 CTAs x 3 x 32 KB bulk-copy ring (the resident kernel's E stream)
//   tiles+pf   : same, each CTA first issues cp.async.bulk.prefetch.L2 for all of its tiles
//   tiles+pf1  : same, but the prefetch runs one tile ahead of the ring only
//   ldg        : plain 16-byte loads, 8 CTAs x 256 threads per SM, 4 loads in flight per thread
//   pf-only    : a kernel that only issues the L2 prefetches, then the tile stream (both timed)
//   wflush     : tiles, with a 512 MB WRITE flush instead (dirty lines evicted during the stream)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stream_prefetch tools/stream_prefetch.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2411_15707_b200/csrc/common.cuh"

using namespace nimbus;

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

// pf: 0 none, 1 all of the CTA's tiles up front, 2 one tile ahead
__global__ void __launch_bounds__(128) k_tiles(const uint8_t* src, uint32_t ntiles, uint32_t tile, uint32_t stages,
                                              uint32_t bytes, int pf, unsigned long long* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bars[16];
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < stages; s++) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (pf == 1) {
        // 128 threads split the CTA's tiles into 32 KB prefetches
        const uint32_t per = tile / 32768;
        uint32_t idx = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x)
            for (uint32_t q = 0; q < per; q++, idx++)
                if (idx % blockDim.x == threadIdx.x) prefetch_l2(src + (size_t)t * tile + (size_t)q * 32768, 32768);
    }
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
            if (pf == 2 && q == 0 && t + gridDim.x < ntiles) prefetch_l2(src + (size_t)(t + gridDim.x) * tile, tile);
            mbar_arrive_expect_tx(&bars[s], bytes);
            bulk_g2s(smem + s * bytes, src + (size_t)t * tile + (size_t)q * bytes, bytes, &bars[s], pol);
            if (++q == per) { q = 0; t += gridDim.x; }
        }
    }
    sink[blockIdx.x] = acc;
}

__global__ void k_pf_only(const uint8_t* src, size_t total) {
    for (size_t o = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 32768; o < total;
         o += (size_t)gridDim.x * blockDim.x * 32768)
        prefetch_l2(src + o, 32768);
}

__global__ void __launch_bounds__(256) k_ldg(const uint4* p, size_t n, unsigned long long* sink) {
    unsigned long long acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        const uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride),
                    d = __ldcs(p + i + 3 * stride);
        acc += a.x ^ b.y ^ c.z ^ d.w;
    }
    for (; i < n; i += stride) acc += p[i].x;
    if (acc == 7) sink[0] = acc;
}

__global__ void k_read(const uint4* p, size_t n, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc += p[i].x;
    if (acc == 7) sink[0] = acc;
}
__global__ void k_write(uint4* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(i, 1, 2, 3);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t mb = 50, total = mb << 20;
    const size_t tile = 96 * 1024, ntiles = total / tile;
    uint8_t *src, *fl;
    cudaMalloc(&src, 8 * total);
    cudaMemset(src, 1, 8 * total);
    cudaMalloc(&fl, (size_t)512 << 20);
    cudaMemset(fl, 2, (size_t)512 << 20);
    unsigned long long* sink;
    cudaMalloc(&sink, 64 * 1024);
    const size_t smem = 3 * 32768 + 1024;
    cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    static const char* names[] = {"tiles", "tiles+pf", "tiles+pf1", "ldg", "pf-only+tiles", "wflush tiles",
                                  "ldg 16/SM", "tiles 2x(3x32K)/SM"};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int pass = 0; pass < 2; pass++)
    for (int mode = 0; mode < 8; mode++) {
        float best = 1e9, sum = 0;
        const int reps = 16;
        for (int rep = 0; rep < reps; rep++) {
            const uint8_t* s = src + (size_t)(rep % 8) * total;
            if (mode == 5) k_write<<<sms * 4, 256>>>(reinterpret_cast<uint4*>(fl), ((size_t)512 << 20) / 16);
            else k_read<<<sms * 4, 256>>>(reinterpret_cast<const uint4*>(fl), ((size_t)512 << 20) / 16, sink);
            cudaEventRecord(e0);
            switch (mode) {
            case 0: case 5: k_tiles<<<sms, 128, smem>>>(s, ntiles, tile, 3, 32768, 0, sink); break;
            case 1: k_tiles<<<sms, 128, smem>>>(s, ntiles, tile, 3, 32768, 1, sink); break;
            case 2: k_tiles<<<sms, 128, smem>>>(s, ntiles, tile, 3, 32768, 2, sink); break;
            case 3: k_ldg<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(s), total / 16, sink); break;
            case 4:
                k_pf_only<<<sms, 32>>>(s, total);
                k_tiles<<<sms, 128, smem>>>(s, ntiles, tile, 3, 32768, 0, sink);
                break;
            case 6: k_ldg<<<sms * 16, 128>>>(reinterpret_cast<const uint4*>(s), total / 16, sink); break;
            case 7: k_tiles<<<sms * 2, 128, smem>>>(s, ntiles, tile, 3, 32768, 0, sink); break;
            }
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep >= 2) { best = ms < best ? ms : best; sum += ms; }
        }
        if (pass == 1)
            printf("%-20s best %6.2f us (%5.0f GB/s) mean %6.2f us  %s\n", names[mode], best * 1e3,
                   (double)total / (best * 1e-3) / 1e9, sum / (reps - 2) * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    // back-to-back: 64 reads of rotating copies timed as one block (no host sync, no flush between;
    // copy i was last read 8 reads = 400 MB earlier, so it is not L2-resident)
    for (int mode = 0; mode < 3; mode++) {
        float best = 1e9;
        for (int rep = 0; rep < 4; rep++) {
            cudaEventRecord(e0);
            for (int i = 0; i < 64; i++) {
                const uint8_t* s = src + (size_t)(i % 8) * total;
                if (mode == 0) k_tiles<<<sms, 128, smem>>>(s, ntiles, tile, 3, 32768, 0, sink);
                else if (mode == 1) k_ldg<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(s), total / 16, sink);
                else k_tiles<<<sms * 2, 128, smem>>>(s, ntiles, tile, 3, 32768, 0, sink);
            }
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        static const char* nm[] = {"b2b tiles", "b2b ldg", "b2b tiles 2/SM"};
        printf("%-20s %6.2f us per 50 MB read (%5.0f GB/s)  %s\n", nm[mode], best * 1e3 / 64,
               (double)total * 64 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    // sizes: single cold read of S MB (ldg), flush before
    for (size_t smb : {25, 50, 100, 200, 400}) {
        uint8_t* big;
        cudaMalloc(&big, smb << 20);
        cudaMemset(big, 3, smb << 20);
        float best = 1e9;
        for (int rep = 0; rep < 6; rep++) {
            k_read<<<sms * 4, 256>>>(reinterpret_cast<const uint4*>(fl), ((size_t)512 << 20) / 16, sink);
            cudaEventRecord(e0);
            k_ldg<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(big), (smb << 20) / 16, sink);
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) best = ms < best ? ms : best;
        }
        printf("cold ldg %4zu MB   %7.2f us (%5.0f GB/s)\n", smb, best * 1e3, (double)(smb << 20) / (best * 1e-3) / 1e9);
        cudaFree(big);
    }
    // empty-kernel event time (launch + event overhead)
    {
        float best = 1e9;
        for (int rep = 0; rep < 10; rep++) {
            cudaEventRecord(e0);
            k_pf_only<<<sms, 32>>>(src, 0);
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("empty kernel       %6.2f us\n", best * 1e3);
    }
    return 0;
}
