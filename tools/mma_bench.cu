// mma_bench.cu -- microbenchmark of tcgen05.mma kind::i8 issue throughput on
// sm_100a as a function of N (M = 128, cta_group::1, both operands in shared
// memory, K-major SWIZZLE_128B).  One CTA per SM issues a long stream of MMAs
// on resident operands; reports cycles per MMA and the implied int8 TOPS.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2411_15707_b200/csrc/common.cuh"

using namespace nimbus;

template <uint32_t N>
__global__ void __launch_bounds__(128, 1) k_mma(uint32_t iters, unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem;                 // 128 rows x 128 B
    uint8_t* B = smem + 16384;         // 256 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    for (uint32_t i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_i8(128, N);
        const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
        long long t0 = clock64();
        for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
            for (uint32_t kk = 0; kk < 4; kk++) {
                mma_i8_ss(tmem + (kk & 1) * 256, sdesc_kmajor_sw128(a0 + kk * 32), sdesc_kmajor_sw128(b0 + kk * 32),
                          idesc, it | kk);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

// A operand from TMEM (columns [256, 288)), B from shared memory; optional
// concurrent bulk-copy fill traffic into a separate shared-memory buffer
// (fill_kb KB per 4 MMAs) to see whether TMA writes compete with MMA reads.
template <uint32_t N, bool TMEM_A, bool MIX = false, bool LD = false>
__global__ void __launch_bounds__(128, 1) k_mma2(uint32_t iters, uint32_t fill_bytes, const uint8_t* gsrc,
                                                 unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem;                 // 128 rows x 128 B
    uint8_t* B = smem + 16384;         // 256 rows x 128 B
    uint8_t* F = smem + 16384 + 32768; // fill target, up to 64 KB
    __shared__ uint64_t bar, fbar;
    __shared__ uint32_t tslot;
    __shared__ volatile uint32_t stop;
    for (uint32_t i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&fbar, 1); stop = 0; fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (TMEM_A && threadIdx.x == 0) {
        for (uint32_t kk = 0; kk < 4; kk++)
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" :: "r"(tmem + 256 + kk * 8),
                         "l"(sdesc_kmajor_sw128(smem_u32(A) + kk * 32)) : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_i8(128, N);
        const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
        long long t0 = clock64();
        for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
            for (uint32_t kk = 0; kk < 4; kk++) {
                if (MIX) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                                 :: "r"(tmem), "r"(tmem + 256 + kk * 8), "l"(sdesc_kmajor_sw128(b0 + kk * 32)),
                                    "r"(idesc), "r"(it | kk) : "memory");
                    mma_i8_ss(tmem + 32, sdesc_kmajor_sw128(a0 + kk * 32), sdesc_kmajor_sw128(b0 + kk * 32), idesc, 1);
                } else if (TMEM_A) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                                 :: "r"(tmem), "r"(tmem + 256 + kk * 8), "l"(sdesc_kmajor_sw128(b0 + kk * 32)),
                                    "r"(idesc), "r"(it | kk) : "memory");
                } else {
                    mma_i8_ss(tmem, sdesc_kmajor_sw128(a0 + kk * 32), sdesc_kmajor_sw128(b0 + kk * 32), idesc, it | kk);
                }
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
        stop = 1;
    } else if (LD && threadIdx.x >= 32) {
        // warps 1-3: continuous TMEM reads (lanes of their subpartition) of columns 384..447
        const uint32_t sub = (threadIdx.x >> 5) & 3;
        uint32_t x = 0;
        while (!stop) {
            uint32_t v[8];
#pragma unroll
            for (int c = 0; c < 8; c++) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                               "=r"(v[7]) : "r"(tmem + ((sub * 32) << 16) + 384 + c * 8));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                x ^= v[0] ^ v[7];
            }
        }
        if (x == 0x1234567) cycles[blockIdx.x] = 0;
    } else if (threadIdx.x == 32 && fill_bytes) {
        uint32_t ph = 0;
        const uint64_t pol = policy_evict_last();
        while (!stop) {
            mbar_arrive_expect_tx(&fbar, fill_bytes);
            bulk_g2s(F, gsrc + (blockIdx.x % 8) * 65536, fill_bytes, &fbar, pol);
            mbar_wait(&fbar, ph);
            ph ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <uint32_t N, bool TMEM_A, bool MIX = false, bool LD = false>
void run2(int sms, uint32_t fill, const uint8_t* g) {
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms);
    const size_t smem = 16384 + 32768 + 65536 + 1024;
    cudaFuncSetAttribute(k_mma2<N, TMEM_A, MIX, LD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint32_t iters = 4096;
    k_mma2<N, TMEM_A, MIX, LD><<<sms, 128, smem>>>(64, fill, g, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_mma2<N, TMEM_A, MIX, LD><<<sms, 128, smem>>>(iters, fill, g, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[256];
    cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < sms; i++) cyc += h[i];
    cyc /= sms;
    const double mmas = 4.0 * iters * (MIX ? 2 : 1);
    printf("%s N=%3u fill=%5u B: %6.1f cycles/MMA (floor %5.1f)  %s\n", MIX ? (LD ? "MIX+LDTM" : "MIX TS+SS") : (TMEM_A ? (LD ? "TMEM-A+LDTM" : "TMEM-A") : (LD ? "SMEM-A+LDTM" : "SMEM-A")), N, fill,
           cyc / mmas, 128.0 * N / 256.0, cudaGetErrorString(err));
    cudaFree(d);
}

template <uint32_t N>
void run(int sms) {
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms);
    const size_t smem = 16384 + 32768 + 1024;
    cudaFuncSetAttribute(k_mma<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint32_t iters = 4096;
    k_mma<N><<<sms, 128, smem>>>(64, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_mma<N><<<sms, 128, smem>>>(iters, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[256];
    cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < sms; i++) cyc += h[i];
    cyc /= sms;
    const double mmas = 4.0 * iters;
    const double ops = 2.0 * 128 * N * 32 * mmas * sms;
    printf("N=%3u  %6.1f cycles/MMA (floor %5.1f)  %7.1f TOPS over %.3f ms  %s\n", N, cyc / mmas, 128.0 * N / 256.0,
           ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(err));
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<64>(sms);
    run<128>(sms);
    run<192>(sms);
    run<256>(sms);
    uint8_t* g;
    cudaMalloc(&g, 1 << 20);
    cudaMemset(g, 1, 1 << 20);
    run2<128, true, true, true>(sms, 0, g);
    run2<128, false, false, true>(sms, 0, g);
    run2<192, false, false, true>(sms, 0, g);
    run2<128, true, false, true>(sms, 0, g);
    for (uint32_t f : {0u, 16384u, 65536u}) {
        run2<128, true, true>(sms, f, g);
        run2<128, false>(sms, f, g);
        run2<128, true>(sms, f, g);
    }
    run2<32, true>(sms, 0, g);
    run2<64, true>(sms, 0, g);
    run2<128, true>(sms, 0, g);
    run2<192, true>(sms, 0, g);
    run2<256, true>(sms, 0, g);
    for (uint32_t f : {4096u, 16384u, 65536u}) {
        run2<192, false>(sms, f, g);
        run2<64, true>(sms, f, g);
        run2<192, true>(sms, f, g);
    }
    return 0;
}
