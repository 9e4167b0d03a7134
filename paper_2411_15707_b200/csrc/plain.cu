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
