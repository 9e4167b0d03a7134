#include <cstdio>
// cop_cc.cu -- K6: the COP contraction on CUDA cores (ablation; first parity
// kernel).  Alg. 1 step 2:
//     C[alpha][col] = sum_beta X[alpha][beta] * E[beta][col]  mod p(col)
// with 32x32->64-bit multiply-adds and lazy reduction: for ell <= 16 every
// product is < 2^47 and m <= 2^17 terms fit in uint64 exactly; for wider X the
// 64-bit sum carries into a 32-bit overflow counter.  One reduction per output.
// Reads the same resident byte-plane Enc(W) as the tensor-core kernel.
#include "internal.h"

namespace nimbus {

constexpr int kCcRows = 8;     // rows (alpha) per thread
constexpr int kCcCols = 128;   // columns per CTA (one per thread)

__device__ __forceinline__ uint32_t assemble(uint32_t p0, uint32_t p1, uint32_t p2, uint32_t p3, uint32_t u) {
    // byte u of each plane word -> E = b0 | b1<<8 | b2<<16 | b3<<24
    const uint32_t sel = u | ((u + 4) << 4);
    const uint32_t lo = __byte_perm(p0, p1, sel);
    const uint32_t hi = __byte_perm(p2, p3, sel);
    return __byte_perm(lo, hi, 0x5410);
}

template <bool WIDE>
__global__ void __launch_bounds__(kCcCols) k_cop_cc(Rns R, const uint8_t* __restrict__ Et,
                                                    const uint32_t* __restrict__ X, uint32_t k, uint32_t m,
                                                    uint32_t KB, uint32_t bn, uint32_t ncol,
                                                    uint32_t* __restrict__ C) {
    __shared__ uint32_t sX[kCcRows][kBK];
    const uint32_t col = blockIdx.x * kCcCols + threadIdx.x;   // ncol is a multiple of 128
    const uint32_t ct = col / bn, r = col % bn;
    const uint32_t alpha0 = blockIdx.y * kCcRows;
    const uint32_t limb = (col / R.N) % R.L, p = R.p[limb];
    const size_t plane = (size_t)bn * kBK;
    uint64_t acc[kCcRows];
    uint32_t carry[kCcRows];
#pragma unroll
    for (int q = 0; q < kCcRows; q++) { acc[q] = 0; carry[q] = 0; }

    for (uint32_t kb = 0; kb < KB; kb++) {
        __syncthreads();
        for (uint32_t idx = threadIdx.x; idx < kCcRows * kBK; idx += kCcCols) {
            const uint32_t rr = idx / kBK, b = idx % kBK, beta = kb * kBK + b, alpha = alpha0 + rr;
            sX[rr][b] = (alpha < k && beta < m) ? X[(size_t)alpha * m + beta] : 0u;
        }
        __syncthreads();
        const uint8_t* tb = Et + ((size_t)ct * KB + kb) * kSW * plane;
#pragma unroll 1
        for (uint32_t c16 = 0; c16 < 8; c16++) {
            const uint32_t off = r * 128u + ((c16 ^ (r & 7u)) << 4);
            const uint4 P0 = __ldg(reinterpret_cast<const uint4*>(tb + 0 * plane + off));
            const uint4 P1 = __ldg(reinterpret_cast<const uint4*>(tb + 1 * plane + off));
            const uint4 P2 = __ldg(reinterpret_cast<const uint4*>(tb + 2 * plane + off));
            const uint4 P3 = __ldg(reinterpret_cast<const uint4*>(tb + 3 * plane + off));
            const uint32_t w0[4] = {P0.x, P0.y, P0.z, P0.w}, w1[4] = {P1.x, P1.y, P1.z, P1.w};
            const uint32_t w2[4] = {P2.x, P2.y, P2.z, P2.w}, w3[4] = {P3.x, P3.y, P3.z, P3.w};
#pragma unroll
            for (int q = 0; q < 4; q++) {
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const uint32_t E = assemble(w0[q], w1[q], w2[q], w3[q], u);
                    const uint32_t bl = c16 * 16 + q * 4 + u;
#pragma unroll
                    for (int rr = 0; rr < kCcRows; rr++) {
                        const uint64_t prod = (uint64_t)sX[rr][bl] * E;
                        acc[rr] += prod;
                        if (WIDE) carry[rr] += (acc[rr] < prod);
                    }
                }
            }
        }
    }
    const uint64_t mu = R.mu[limb];
    const uint32_t two64 = WIDE ? mulmod(mod64(1ULL << 32, p, mu), mod64(1ULL << 32, p, mu), p, mu) : 0;
#pragma unroll
    for (int rr = 0; rr < kCcRows; rr++) {
        const uint32_t alpha = alpha0 + rr;
        if (alpha >= k) break;
        uint32_t v = mod64(acc[rr], p, mu);
        if (WIDE) v = addmod(v, mulmod(carry[rr] % p, two64, p, mu), p);
        C[(size_t)alpha * ncol + col] = v;
    }
}

cudaError_t launch_cop_cudacore(nimbus_ctx* c, const nimbus_encw* w, const uint32_t* d_X, uint32_t k,
                                uint32_t* d_C, cudaStream_t st) {
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    dim3 g(ncol / kCcCols, (k + kCcRows - 1) / kCcRows);
    if (c->rns.ell <= 16)
        k_cop_cc<false><<<g, kCcCols, 0, st>>>(c->rns, w->d_Et, d_X, k, w->m, w->KB, w->bn, ncol, d_C);
    else
        k_cop_cc<true><<<g, kCcCols, 0, st>>>(c->rns, w->d_Et, d_X, k, w->m, w->KB, w->bn, ncol, d_C);
    c->launches++;
    snprintf(c->last_contraction, sizeof(c->last_contraction), "k_cop_cc");
    return cudaGetLastError();
}

}  // namespace nimbus
