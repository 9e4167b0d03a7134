// gen_a_rate.cu -- how fast can the SMs regenerate the `a` half of Enc(W)
// (a_i[beta][j] = uniform_mod(word(seed, 2, (beta L + i) N + j), p_i), App. B)
// straight into the contraction's K-major SW128 byte-plane smem layout?
// C2 shape: m = 768 rows, L = 2, N = 4096 -> 6.29 M residues.  One unit =
// 16 consecutive beta of one column -> 4 x 16-byte plane stores.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gen_a_rate tools/gen_a_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2411_15707_b200/csrc/common.cuh"

using namespace nimbus;

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_gen(uint64_t key, uint32_t m, uint32_t L, uint32_t N, uint32_t p0,
                                                 uint32_t p1, uint32_t BN, unsigned long long* sink) {
    __shared__ __align__(1024) uint8_t slot[4 * 32 * 256];     // 4 planes x 32 cols x 256 B (2 k-blocks)
    const uint32_t ncolA = L * N, tiles = ncolA / BN;
    const uint32_t kpairs = (m + 255) / 256;
    const uint64_t step = 0x9E3779B97F4A7C15ULL * (uint64_t)L * N;
    for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (uint32_t kp = 0; kp < kpairs; kp++) {
            // 32 cols x 16 chunks of 16 beta
            for (uint32_t u = threadIdx.x; u < BN * 16; u += THREADS) {
                const uint32_t c = u >> 4, ch = u & 15;
                const uint32_t col = t * BN + c;
                const uint32_t limb = col / N, j = col - limb * N;
                const uint32_t p = limb ? p1 : p0;
                const uint32_t b0 = kp * 256 + ch * 16;
                uint64_t x = key + 0x9E3779B97F4A7C15ULL * (((uint64_t)b0 * L + limb) * N + j + 1);
                uint32_t w[4][4];
#pragma unroll
                for (int r = 0; r < 16; r++) {
                    const uint32_t a = samp_uniform_mod(mix64(x), p);
                    x += step;
                    // byte plane s gets byte s of a; 4 residues per 32-bit word
#pragma unroll
                    for (int s = 0; s < 4; s++) {
                        const uint32_t bt = (a >> (8 * s)) & 0xFF;
                        if ((r & 3) == 0) w[s][r >> 2] = bt;
                        else w[s][r >> 2] |= bt << (8 * (r & 3));
                    }
                }
                const uint32_t kb = ch >> 3, q = ch & 7;
#pragma unroll
                for (int s = 0; s < 4; s++) {
                    uint8_t* dst = slot + (kb * 4 + s) * (32 * 128) + c * 128;   // [kb][plane][col][128 B]
                    *reinterpret_cast<uint4*>(dst + ((q ^ (c & 7)) << 4)) = make_uint4(w[s][0], w[s][1], w[s][2], w[s][3]);
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) sink[blockIdx.x] = slot[blockIdx.x & 1023];
}

template <int T>
static void run(int sms, int ctas_per_sm, unsigned long long* sink) {
    const uint32_t m = 768, L = 2, N = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 10; rep++) {
        cudaEventRecord(e0);
        k_gen<T><<<sms * ctas_per_sm, T>>>(0x1234567ULL, m, L, N, 2147377153u, 2147352577u, 32, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double res = (double)m * L * N;
    printf("threads %3d x %d CTA/SM: %.2f us for %.2f M residues (%.2f Gres/s)  %s\n", T, ctas_per_sm, best * 1e3,
           res / 1e6, res / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* sink;
    cudaMalloc(&sink, 1 << 20);
    run<128>(sms, 1, sink);
    run<256>(sms, 1, sink);
    run<512>(sms, 1, sink);
    run<256>(sms, 2, sink);
    run<512>(sms, 2, sink);
    return 0;
}
