// plain.cu -- server side of Alg. 1 step 5: the server's local
// product W<X>_s, i.e. Y = X.W mod 2^ell on plaintext shares, and the
// combination <Y>_s = X_s.W + unpack(Dec(c)) mod 2^ell.
//
// X.W mod 2^ell is an exact integer GEMM.  With 8-bit slices X = sum_i x_i 2^(8i),
// W = sum_j w_j 2^(8j) (S = S_x slices each, the same slicing as the COP
// contraction), X.W = sum_s 2^(8s) acc_s with acc_s = sum_{i+j=s} x_i.w_j, and
// only shifts 8s < ell survive mod 2^ell: s < S.  acc_s is exact in int32 up to
// m <= 2^31 / (S 255^2); beyond that int32 wrap-around is harmless because
// every acc_s is needed only mod 2^32 (2^(8s) acc_s mod 2^ell, ell <= 32).
//
// Layout: plaintext W in tcgen05 B-operand tiles, Wt[ct][kb][j < S][64 rows = columns][128 B of beta],
// swizzled like Enc(W) (layout.cu); X slices from k_slice_x.  Kernel k_plain_tc: persistent,
// warp 0 bulk-copy producer (X slices + W planes per k-block), warp 1 MMA issuer, warps 4-11 epilogue.
// For slice i one MMA with the W planes 0..S-1-i stacked along N writes x_i w_j into
// acc_{i+j} (D at TMEM column 64 i): S(S+1)/2 plane products instead of S^2.
#include "slice_dev.cuh"

namespace nimbus {

constexpr uint32_t kBNP = 64;   // output columns per W tile

// ---------------------------------------------------------------- tile plaintext W
// CTA (ct, kb): W[beta][col] (row-major m x n) -> S byte planes Wt[ct][kb][j][64][128 B swizzled]
template <int S>
__global__ void __launch_bounds__(256) k_tile_plainw(const uint32_t* __restrict__ W, uint32_t m, uint32_t n,
                                                     uint32_t KB, uint8_t* __restrict__ Wt) {
    __shared__ uint32_t sW[kBK][kBNP + 1];
    const uint32_t ct = blockIdx.x, kb = blockIdx.y;
    for (uint32_t idx = threadIdx.x; idx < kBK * kBNP; idx += blockDim.x) {
        const uint32_t b = idx / kBNP, c = idx % kBNP, beta = kb * kBK + b, col = ct * kBNP + c;
        sW[b][c] = (beta < m && col < n) ? W[(size_t)beta * n + col] : 0u;
    }
    __syncthreads();
    uint8_t* base = Wt + ((size_t)ct * KB + kb) * S * kBNP * kBK;
    for (uint32_t idx = threadIdx.x; idx < S * kBNP * 8; idx += blockDim.x) {
        const uint32_t j = idx / (kBNP * 8), r = (idx / 8) % kBNP, c16 = idx % 8;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint32_t acc = 0;
#pragma unroll
            for (int u = 0; u < 4; u++) acc |= ((sW[c16 * 16 + 4 * q + u][r] >> (8 * j)) & 0xFF) << (8 * u);
            w[q] = acc;
        }
        *reinterpret_cast<uint4*>(base + (size_t)j * kBNP * kBK + swz_off(r, c16)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ---------------------------------------------------------------- plain GEMM mod 2^ell
template <int S>
struct PlainCfg {
    static constexpr uint32_t BM = kBM, BN = kBNP, BK = kBK;
    static constexpr uint32_t A_BYTES = S * BM * BK;      // X slices
    static constexpr uint32_t B_BYTES = S * BN * BK;      // W planes
    static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
    static constexpr uint32_t STAGES = (200u * 1024u) / STAGE > 6 ? 6 : (200u * 1024u) / STAGE;
    static constexpr uint32_t ACC_COLS = S * BN;          // acc_0 .. acc_{S-1}
    static constexpr uint32_t BUF_STRIDE = 256;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr uint32_t EPI_WARPS = 8;
    static constexpr uint32_t THREADS = 128 + 32 * EPI_WARPS;
    static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 256;
    static_assert(ACC_COLS <= BUF_STRIDE, "two accumulator sets must fit in TMEM");
    static_assert(SMEM <= 232448, "shared memory");
};

// Y[row][col] = (sum_s acc_s 2^(8s) + add[row][col]) mod 2^ell for row < k, col < n
template <int S>
__global__ void __launch_bounds__(PlainCfg<S>::THREADS, 1)
k_plain_tc(const uint8_t* __restrict__ Xt, const uint8_t* __restrict__ Wt, uint32_t k, uint32_t n, uint32_t Mt,
           uint32_t CT, uint32_t KB, uint32_t ell, const uint32_t* __restrict__ add, uint32_t* __restrict__ Y) {
    using Cfg = PlainCfg<S>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nunits = Mt * CT;
    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (uint32_t b = 0; b < 2; b++) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], Cfg::EPI_WARPS); }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer
            const uint64_t pol_a = policy_evict_last();    // X slices: reused by every column tile
            const uint64_t pol_b = policy_evict_first();   // W planes: streamed
            uint32_t it = 0;
            bool waited = false;
            for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x) {
                const uint32_t mt = u % Mt, ct = u / Mt;
                for (uint32_t kb = 0; kb < KB; kb++, it++) {
                    const uint32_t s = it % Cfg::STAGES, ph = (it / Cfg::STAGES) & 1;
                    if (it >= Cfg::STAGES) mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* sa = smem + s * Cfg::STAGE;
                    mbar_arrive_expect_tx(&full[s], Cfg::STAGE);
                    bulk_g2s(sa + Cfg::A_BYTES, Wt + ((size_t)ct * KB + kb) * Cfg::B_BYTES, Cfg::B_BYTES, &full[s],
                             pol_b);
                    if (!waited) { pdl_wait(); waited = true; }     // X slices come from the slice kernel
                    bulk_g2s(sa, Xt + ((size_t)mt * KB + kb) * Cfg::A_BYTES, Cfg::A_BYTES, &full[s], pol_a);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer: slice i x planes 0..S-1-i -> acc_i .. acc_{S-1}
            uint32_t it = 0, ti = 0;
            for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ti++) {
                const uint32_t buf = ti & 1, use = ti >> 1;
                if (ti >= 2) mbar_wait(&tempty[buf], (use & 1) ^ 1);
                tc_fence_after();
                const uint32_t dacc = tmem + buf * Cfg::BUF_STRIDE;
                for (uint32_t kb = 0; kb < KB; kb++, it++) {
                    const uint32_t s = it % Cfg::STAGES, ph = (it / Cfg::STAGES) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(smem + s * Cfg::STAGE);
                    const uint32_t b0 = a0 + Cfg::A_BYTES;
#pragma unroll
                    for (uint32_t kk = 0; kk < Cfg::BK / 32; kk++) {
                        const uint64_t bd = sdesc_kmajor_sw128(b0 + kk * 32);
#pragma unroll
                        for (uint32_t i = 0; i < (uint32_t)S; i++) {
                            const uint64_t ad = sdesc_kmajor_sw128(a0 + i * Cfg::BM * Cfg::BK + kk * 32);
                            // i = 0 writes every acc_s (fresh at the first k-step); i >= 1 adds into them
                            mma_i8_ss(dacc + i * Cfg::BN, ad, bd, idesc_i8(Cfg::BM, (S - i) * Cfg::BN),
                                      (i > 0 || (kb | kk) != 0) ? 1u : 0u);
                        }
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&tfull[buf]);
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: row = TMEM lane, 8 columns per tcgen05.ld, half the tile per warp
        const uint32_t ew = warp - 4;
        const uint32_t sub = ew & 3, half = ew >> 2;
        const uint32_t tmask = ell >= 32 ? 0xFFFFFFFFu : ((1u << ell) - 1u);
        uint32_t ti = 0;
        for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ti++) {
            const uint32_t mt = u % Mt, ct = u / Mt;
            const uint32_t buf = ti & 1, use = ti >> 1;
            mbar_wait(&tfull[buf], use & 1);
            tc_fence_after();
            const uint32_t row = mt * Cfg::BM + sub * 32 + lane;
            const uint32_t tacc = tmem + ((sub * 32) << 16) + buf * Cfg::BUF_STRIDE;
#pragma unroll 1
            for (uint32_t c = 0; c < Cfg::BN / 16; c++) {
                const uint32_t cc = half * (Cfg::BN / 16) + c;       // 8-column chunk of the tile
                uint32_t v[S][8];
#pragma unroll
                for (int s = 0; s < S; s++) tmem_ld8(tacc + s * Cfg::BN + cc * 8, v[s]);
                tmem_ld_wait();
                const uint32_t col0 = ct * Cfg::BN + cc * 8;
                if (row >= k || col0 >= n) continue;
                uint32_t y[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    uint32_t x = v[0][q];
#pragma unroll
                    for (int s = 1; s < S; s++) x += v[s][q] << (8 * s);    // mod 2^32
                    y[q] = x;
                }
                const size_t o = (size_t)row * n + col0;
                if (col0 + 8 <= n && (n & 3) == 0) {
                    if (add) {
                        const uint4 a0 = *reinterpret_cast<const uint4*>(add + o);
                        const uint4 a1 = *reinterpret_cast<const uint4*>(add + o + 4);
                        y[0] += a0.x; y[1] += a0.y; y[2] += a0.z; y[3] += a0.w;
                        y[4] += a1.x; y[5] += a1.y; y[6] += a1.z; y[7] += a1.w;
                    }
#pragma unroll
                    for (int q = 0; q < 8; q++) y[q] &= tmask;
                    *reinterpret_cast<uint4*>(Y + o) = make_uint4(y[0], y[1], y[2], y[3]);
                    *reinterpret_cast<uint4*>(Y + o + 4) = make_uint4(y[4], y[5], y[6], y[7]);
                } else {
#pragma unroll
                    for (int q = 0; q < 8; q++)
                        if (col0 + q < n) Y[o + q] = (y[q] + (add ? add[o + q] : 0u)) & tmask;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, Cfg::TMEM_COLS);
    }
}

// ---------------------------------------------------------------- ell = 64 (the paper's t)
// X.W mod 2^64 with 8 slices of each operand: acc_s = sum_{i+j=s} x_i w_j for s < 8 only
// (shifts 8s >= 64 vanish mod 2^64): 36 of the 64 slice products.  acc_s < 8 m 255^2 < 2^31
// for m <= 4096 (host-checked), so Y = sum_s acc_s 2^(8s) in 64-bit wrap-around is exact mod 2^64.
// Transposed orientation (as the COP kernel k_cop_tc_t<8>): A = the 8 byte planes of a
// 128-column W tile (M = 128 output columns), B = the 8 X slices of a 32-row tile stacked along
// N; plane j multiplies only slices 0 .. 7-j (N = 32 (8 - j)), D at TMEM column 32 j, so it
// writes exactly acc_j .. acc_7.  Plane 0's first MMA (N = 256) initialises all 8 accumulators.
// Shared memory: 2 X slots (32 KB) + 4 plane-quad slots (64 KB) = 192 KB; TMEM: 2 sets x 256.
constexpr uint32_t kBNP64 = 128;   // output columns per W tile at ell = 64

// CTA (ct, kb): W[beta][col] uint64 -> 8 byte planes Wt[ct][kb][j][128 rows = columns][128 B swizzled].
// Thread item (16-byte chunk c16, column r; r fastest: coalesced W reads) reads 16 entries once and
// writes the chunk of every plane.
__global__ void __launch_bounds__(256) k_tile_plainw64(const uint64_t* __restrict__ W, uint32_t m, uint32_t n,
                                                       uint32_t KB, uint8_t* __restrict__ Wt) {
    const uint32_t ct = blockIdx.x, kb = blockIdx.y;
    uint8_t* base = Wt + ((size_t)ct * KB + kb) * 8 * kBNP64 * kBK;
    for (uint32_t idx = threadIdx.x; idx < 8 * kBNP64; idx += blockDim.x) {
        const uint32_t r = idx % kBNP64, c16 = idx / kBNP64, col = ct * kBNP64 + r;
        uint64_t v[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const uint32_t beta = kb * kBK + c16 * 16 + u;
            v[u] = (beta < m && col < n) ? W[(size_t)beta * n + col] : 0ull;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                uint32_t acc = 0;
#pragma unroll
                for (int u = 0; u < 4; u++) acc |= (uint32_t)((v[4 * q + u] >> (8 * j)) & 0xFF) << (8 * u);
                w[q] = acc;
            }
            *reinterpret_cast<uint4*>(base + (size_t)j * kBNP64 * kBK + swz_off(r, c16)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

struct Plain64Cfg {
    static constexpr uint32_t BM = kBNP64, RT = 32, BK = kBK;
    static constexpr uint32_t X_BYTES = 8 * RT * BK;        // 32 KB: 8 slices x 32 rows
    static constexpr uint32_t Q_BYTES = 4 * BM * BK;        // 64 KB: 4 planes
    static constexpr uint32_t OFF_Q = 2 * X_BYTES;
    static constexpr uint32_t RING = OFF_Q + 2 * Q_BYTES;
    static constexpr uint32_t EPI_WARPS = 8;
    static constexpr uint32_t THREADS = 128 + 32 * EPI_WARPS;
    static constexpr size_t SMEM = (size_t)RING + 1024 + 256;
    static_assert(SMEM <= 232448, "shared memory");
};

// Y[row][col] = (sum_{s<8} acc_s 2^(8s) + add[row][col]) mod 2^64 for row < k, col < n
__global__ void __launch_bounds__(Plain64Cfg::THREADS, 1)
k_plain_t64(const uint8_t* __restrict__ Xt, const uint8_t* __restrict__ Wt, uint32_t k, uint32_t n, uint32_t Mt,
            uint32_t CT, uint32_t KB, const uint64_t* __restrict__ add, uint64_t* __restrict__ Y) {
    using Cfg = Plain64Cfg;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* xfull = reinterpret_cast<uint64_t*>(smem + Cfg::RING);
    uint64_t* xempty = xfull + 2;
    uint64_t* qfull = xempty + 2;
    uint64_t* qempty = qfull + 2;
    uint64_t* tfull = qempty + 2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nunits = Mt * CT;
    if (warp == 0 && lane == 0) {
        for (uint32_t b = 0; b < 2; b++) {
            mbar_init(&xfull[b], 1); mbar_init(&xempty[b], 1); mbar_init(&qfull[b], 1); mbar_init(&qempty[b], 1);
            mbar_init(&tfull[b], 1); mbar_init(&tempty[b], Cfg::EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer: per k-block the X block, then the two plane quads
            const uint64_t pol = policy_evict_last();
            pdl_wait();
            uint32_t ix = 0, iq = 0;
            for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x) {
                const uint32_t mt = u % Mt, ct = u / Mt;
                for (uint32_t kb = 0; kb < KB; kb++) {
                    {
                        const uint32_t s = ix & 1;
                        if (ix >= 2) mbar_wait(&xempty[s], ((ix >> 1) & 1) ^ 1);
                        ix++;
                        mbar_arrive_expect_tx(&xfull[s], Cfg::X_BYTES);
                        bulk_g2s(smem + s * Cfg::X_BYTES, Xt + ((size_t)mt * KB + kb) * Cfg::X_BYTES, Cfg::X_BYTES,
                                 &xfull[s], pol);
                    }
                    for (uint32_t qd = 0; qd < 2; qd++, iq++) {
                        const uint32_t s = iq & 1;
                        if (iq >= 2) mbar_wait(&qempty[s], ((iq >> 1) & 1) ^ 1);
                        mbar_arrive_expect_tx(&qfull[s], Cfg::Q_BYTES);
                        bulk_g2s(smem + Cfg::OFF_Q + s * Cfg::Q_BYTES,
                                 Wt + ((size_t)ct * KB + kb) * 8 * Cfg::BM * Cfg::BK + qd * Cfg::Q_BYTES, Cfg::Q_BYTES,
                                 &qfull[s], pol);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (converged warp): plane j x slices 0..7-j -> acc_j .. acc_7
        const uint64_t x_desc0 = sdesc_kmajor_sw128(smem_u32(smem));
        const uint64_t q_desc0 = sdesc_kmajor_sw128(smem_u32(smem + Cfg::OFF_Q));
        uint32_t ix = 0, iq = 0, ti = 0;
        for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ti++) {
            const uint32_t buf = ti & 1, use = ti >> 1;
            if (ti >= 2) mbar_wait(&tempty[buf], (use & 1) ^ 1);
            tc_fence_after();
            const uint32_t dacc = tmem + buf * 256;
            for (uint32_t kb = 0; kb < KB; kb++, ix++) {
                const uint32_t xs = ix & 1;
                mbar_wait(&xfull[xs], (ix >> 1) & 1);
                const uint64_t bd = x_desc0 + xs * (Cfg::X_BYTES >> 4);
                for (uint32_t qd = 0; qd < 2; qd++, iq++) {
                    const uint32_t qs = iq & 1;
                    mbar_wait(&qfull[qs], (iq >> 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (uint32_t jl = 0; jl < 4; jl++) {
                        const uint32_t j = qd * 4 + jl;
                        const uint64_t ad = q_desc0 + qs * (Cfg::Q_BYTES >> 4) + jl * ((Cfg::BM * Cfg::BK) >> 4);
                        const uint32_t idesc = idesc_i8(Cfg::BM, (8 - j) * Cfg::RT);
#pragma unroll
                        for (uint32_t kk = 0; kk < Cfg::BK / 32; kk++)
                            mma_i8_ss_w(dacc + j * Cfg::RT, ad + 2 * kk, bd + 2 * kk, idesc,
                                        (kb == 0 && kk == 0 && j == 0) ? 0u : 1u);
                    }
                    mma_commit_w(&qempty[qs]);
                }
                mma_commit_w(&xempty[xs]);
            }
            mma_commit_w(&tfull[buf]);
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: lane = output column, 8 rows per tcgen05.ld, 16 rows per warp
        const uint32_t ew = warp - 4;
        const uint32_t sub = ew & 3, half = ew >> 2;
        pdl_wait();
        uint32_t ti = 0;
        for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ti++) {
            const uint32_t mt = u % Mt, ct = u / Mt;
            const uint32_t buf = ti & 1, use = ti >> 1;
            mbar_wait(&tfull[buf], use & 1);
            tc_fence_after();
            const uint32_t col = ct * Cfg::BM + sub * 32 + lane;
            const uint32_t tb = tmem + ((sub * 32) << 16) + buf * 256;
#pragma unroll 1
            for (uint32_t ch = 0; ch < 2; ch++) {
                const uint32_t r0 = half * 16 + ch * 8;
                uint32_t v[8][8];
#pragma unroll
                for (uint32_t s2 = 0; s2 < 8; s2++) tmem_ld8(tb + s2 * Cfg::RT + r0, v[s2]);
                tmem_ld_wait();
#pragma unroll
                for (uint32_t q = 0; q < 8; q++) {
                    const uint32_t row = mt * Cfg::RT + r0 + q;
                    uint64_t y = 0;
#pragma unroll
                    for (uint32_t s2 = 0; s2 < 8; s2++) y += (uint64_t)v[s2][q] << (8 * s2);   // mod 2^64
                    if (row < k && col < n) {
                        const size_t o = (size_t)row * n + col;
                        Y[o] = y + (add ? add[o] : 0ull);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

uint32_t plain_col_tiles64(uint32_t n) { return (n + kBNP64 - 1) / kBNP64; }

cudaError_t launch_tile_plainw64(nimbus_ctx* c, const uint64_t* d_W, uint32_t m, uint32_t n, uint32_t KB,
                                 uint8_t* d_Wt, cudaStream_t st) {
    k_tile_plainw64<<<dim3(plain_col_tiles64(n), KB), 256, 0, st>>>(d_W, m, n, KB, d_Wt);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_plain_matmul64(nimbus_ctx* c, const uint8_t* d_Xt, const uint8_t* d_Wt, uint32_t k, uint32_t n,
                                  uint32_t KB, const uint64_t* d_add, uint64_t* d_Y, cudaStream_t st) {
    using Cfg = Plain64Cfg;
    cudaError_t e = ensure_smem(c, k_plain_t64, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t Mt = (k + Cfg::RT - 1) / Cfg::RT, CT = plain_col_tiles64(n);
    const uint32_t units = Mt * CT;
    const uint32_t grid = units < (uint32_t)c->num_sms ? units : (uint32_t)c->num_sms;
    e = launch_pdl(k_plain_t64, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM, st, d_Xt, d_Wt, k, n, Mt, CT, KB, d_add, d_Y);
    c->launches++;
    {   // writes Y and triggers its dependents early
        const void* op[1] = {d_Y};
        const size_t ob[1] = {(size_t)k * n * 8};
        pdl_outputs_set(st, op, ob, 1);
    }
    return e;
}

// ---------------------------------------------------------------- launchers
uint32_t plain_col_tiles(uint32_t n) { return (n + kBNP - 1) / kBNP; }

cudaError_t launch_tile_plainw(nimbus_ctx* c, const uint32_t* d_W, uint32_t m, uint32_t n, uint32_t KB,
                               uint8_t* d_Wt, cudaStream_t st) {
    const dim3 g(plain_col_tiles(n), KB);
    switch (sx_of(c->rns.ell)) {
        case 1: k_tile_plainw<1><<<g, 256, 0, st>>>(d_W, m, n, KB, d_Wt); break;
        case 2: k_tile_plainw<2><<<g, 256, 0, st>>>(d_W, m, n, KB, d_Wt); break;
        default: k_tile_plainw<4><<<g, 256, 0, st>>>(d_W, m, n, KB, d_Wt); break;
    }
    c->launches++;
    return cudaGetLastError();
}

template <int S>
static cudaError_t launch_plain_s(nimbus_ctx* c, const uint8_t* d_Xt, const uint8_t* d_Wt, uint32_t k, uint32_t n,
                                  uint32_t KB, const uint32_t* d_add, uint32_t* d_Y, cudaStream_t st) {
    using Cfg = PlainCfg<S>;
    {
        cudaError_t e = ensure_smem(c, k_plain_tc<S>, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    const uint32_t Mt = (k + kBM - 1) / kBM, CT = plain_col_tiles(n);
    const uint32_t units = Mt * CT;
    const uint32_t grid = units < (uint32_t)c->num_sms ? units : (uint32_t)c->num_sms;
    {   // writes Y and triggers its dependents early
        const void* op[1] = {d_Y};
        const size_t ob[1] = {(size_t)k * n * 4};
        pdl_outputs_set(st, op, ob, 1);
    }
    return launch_pdl(k_plain_tc<S>, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM, st, d_Xt, d_Wt, k, n, Mt, CT, KB,
                      c->rns.ell, d_add, d_Y);
}

cudaError_t launch_plain_matmul(nimbus_ctx* c, const uint8_t* d_Xt, const uint8_t* d_Wt, uint32_t k, uint32_t n,
                                uint32_t KB, const uint32_t* d_add, uint32_t* d_Y, cudaStream_t st) {
    cudaError_t e;
    switch (sx_of(c->rns.ell)) {
        case 1: e = launch_plain_s<1>(c, d_Xt, d_Wt, k, n, KB, d_add, d_Y, st); break;
        case 2: e = launch_plain_s<2>(c, d_Xt, d_Wt, k, n, KB, d_add, d_Y, st); break;
        default: e = launch_plain_s<4>(c, d_Xt, d_Wt, k, n, KB, d_add, d_Y, st); break;
    }
    c->launches++;
    return e;
}

}  // namespace nimbus
