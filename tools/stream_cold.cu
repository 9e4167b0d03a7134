// stream_cold.cu -- cold (not L2-resident) 50 MB read with the Enc(W) tile
// pattern (CTA c streams 96 KB tiles c, c + grid, ...), swept over copy size,
// copies in flight per CTA and CTAs per SM: what does the resident contraction's
// E stream (3 x 32 KB in flight, one CTA per SM, ~17 us for 50 MB) leave on the
// table?  L2 is made cold by reading (not writing) 512 MB before every run.
// Result on B200 (TILE_KB=384, all copy sizes dividing the tile): ~13.2 us
// (~3.97 TB/s) for 32 KB x 4, 64 KB x 2 or 96 KB x 2 alike -- no copy size or
// depth beats the 3 x 32 KB ring for a cold 50 MB stream.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stream_cold tools/stream_cold.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2411_15707_b200/csrc/common.cuh"

using namespace nimbus;

__device__ __forceinline__ unsigned long long gt_ns() {
    unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}
// hold: SM cycles a landed slot is kept before it is refilled (emulates the MMAs that consume it;
// globaltimer ticks in ~1 us steps here, too coarse)
__global__ void __launch_bounds__(128) k_tiles(const uint8_t* src, uint32_t ntiles, uint32_t tile, uint32_t stages,
                                              uint32_t bytes, unsigned long long* sink, uint32_t hold = 0) {
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
            if (hold) { const long long t0 = clock64(); while (clock64() - t0 < (long long)hold) { } }
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

// contiguous variant: CTA c streams bytes [c*chunk, (c+1)*chunk) in `bytes` copies
__global__ void __launch_bounds__(128) k_contig(const uint8_t* src, size_t total, uint32_t stages, uint32_t bytes,
                                               unsigned long long* sink) {
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
    const size_t ncopies = total / bytes;
    const size_t per = (ncopies + gridDim.x - 1) / gridDim.x;
    const size_t c0 = blockIdx.x * per, c1 = c0 + per < ncopies ? c0 + per : ncopies;
    const uint32_t n = c1 > c0 ? (uint32_t)(c1 - c0) : 0;
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
            bulk_g2s(smem + s * bytes, src + (c0 + i) * bytes, bytes, &bars[s], pol);
        }
    }
    sink[blockIdx.x] = acc;
}

// touch one 16-byte word every `stride` bytes (TLB warm-up; brings < 0.1 % of the lines into L2)
__global__ void k_touch(const uint8_t* p, size_t total, size_t stride, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (size_t o = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * stride; o < total;
         o += (size_t)gridDim.x * blockDim.x * stride)
        acc += *reinterpret_cast<const unsigned long long*>(p + o);
    if (acc == 7) sink[0] = acc;
}

__global__ void k_read(const uint4* p, size_t n, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc += p[i].x;
    if (acc == 7) sink[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t mb = getenv("MB") ? (size_t)atoi(getenv("MB")) : 50;
    const size_t tile = getenv("TILE_KB") ? (size_t)atoi(getenv("TILE_KB")) * 1024 : 96 * 1024;
    const size_t ntiles = (mb << 20) / tile;
    printf("tile %zu KB\n", tile / 1024);
    uint8_t *src, *fl;
    cudaMalloc(&src, (size_t)8 * (mb << 20));   // 8 copies, rotated like bench.py --l2 rotate
    cudaMemset(src, 1, (size_t)8 * (mb << 20));
    cudaMalloc(&fl, (size_t)512 << 20);
    cudaMemset(fl, 2, (size_t)512 << 20);
    unsigned long long* sink;
    cudaMalloc(&sink, 64 * 1024);
    struct V { uint32_t bytes, stages, ctas_per_sm; };
    const V vs[] = {{32768, 3, 1}, {32768, 4, 1}, {32768, 5, 1}, {32768, 6, 1}, {16384, 8, 1}, {16384, 12, 1},
                    {65536, 1, 1}, {65536, 2, 1}, {65536, 3, 1}, {65536, 1, 2}, {49152, 2, 1}, {49152, 4, 1},
                    {98304, 1, 1}, {98304, 2, 1}};
    for (const V& v : vs) {
        const size_t smem = (size_t)v.stages * v.bytes + 1024;
        if (smem * v.ctas_per_sm > 228 * 1024 || tile % v.bytes) continue;   // copies must tile the tile
        cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const uint32_t grid = sms * v.ctas_per_sm;
        float best = 1e9, sum = 0;
        const int reps = 8;
        for (int rep = 0; rep < reps; rep++) {
            k_read<<<sms * 4, 256>>>(reinterpret_cast<const uint4*>(fl), ((size_t)512 << 20) / 16, sink);
            const uint8_t* s = src + (size_t)(rep % 8) * (mb << 20);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_tiles<<<grid, 128, smem>>>(s, (uint32_t)ntiles, (uint32_t)tile, v.stages, v.bytes, sink);
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
            sum += ms;
        }
        printf("%5u B x %2u stages x %u CTA/SM (%4u KB in flight/SM): best %6.2f us (%5.0f GB/s), mean %6.2f us  %s\n",
               v.bytes, v.stages, v.ctas_per_sm, v.bytes * v.stages * v.ctas_per_sm / 1024, best * 1e3,
               (double)ntiles * tile / (best * 1e-3) / 1e9, sum / reps * 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    if (getenv("HOLD_NS")) {
        // the resident kernel's ring with its MMA hold per 32 KB slot: 3, 4, 6 slots
        const uint32_t hold = (uint32_t)atoi(getenv("HOLD_NS"));
        for (uint32_t st : {3u, 4u, 6u}) {
            const size_t smem = (size_t)st * 32768 + 1024;
            cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            float best = 1e9;
            for (int rep = 0; rep < 8; rep++) {
                k_read<<<sms * 4, 256>>>(reinterpret_cast<const uint4*>(fl), ((size_t)512 << 20) / 16, sink);
                const uint8_t* s = src + (size_t)(rep % 8) * (mb << 20);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                k_tiles<<<sms, 128, smem>>>(s, (uint32_t)ntiles, (uint32_t)tile, st, 32768, sink, hold);
                cudaEventRecord(e1);
                cudaDeviceSynchronize();
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("hold %u cycles, %u x 32 KB: best %6.2f us (%5.0f GB/s)\n", hold, st, best * 1e3,
                   (double)ntiles * tile / (best * 1e-3) / 1e9);
        }
    }
    // TLB / pattern experiments at 32 KB x 3 (the resident kernel's ring)
    cudaFuncSetAttribute(k_contig, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768 + 1024);
    cudaFuncSetAttribute(k_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768 + 1024);
    for (int mode = 0; mode < 6; mode++) {
        // 0 tiles, 1 tiles + touch/2MB, 2 tiles + touch/64KB, 3 contiguous, 4 contiguous + touch/2MB, 5 tiles after a warm run
        float best = 1e9, sum = 0;
        const int reps = 8;
        for (int rep = 0; rep < reps; rep++) {
            const uint8_t* s = src + (size_t)(rep % 8) * (mb << 20);
            k_read<<<sms * 4, 256>>>(reinterpret_cast<const uint4*>(fl), ((size_t)512 << 20) / 16, sink);
            if (mode == 1 || mode == 4) k_touch<<<sms, 128>>>(s, mb << 20, (size_t)2 << 20, sink);
            if (mode == 2) k_touch<<<sms, 128>>>(s, mb << 20, (size_t)64 << 10, sink);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (mode >= 3 && mode <= 4) k_contig<<<sms, 128, 3 * 32768 + 1024>>>(s, ntiles * tile, 3, 32768, sink);
            else k_tiles<<<sms, 128, 3 * 32768 + 1024>>>(s, (uint32_t)ntiles, (uint32_t)tile, 3, 32768, sink);
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
            sum += ms;
        }
        static const char* names[] = {"tiles", "tiles+touch2MB", "tiles+touch64KB", "contig", "contig+touch2MB", "-"};
        if (mode < 5)
            printf("%-18s best %6.2f us mean %6.2f us  %s\n", names[mode], best * 1e3, sum / reps * 1e3,
                   cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
