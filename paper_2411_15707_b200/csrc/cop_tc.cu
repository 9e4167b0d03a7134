// cop_tc.cu -- K5: the COP contraction on 5th-generation tensor cores.
//
// Alg. 1 step 2 is the dense modular contraction
//     C[alpha][col] = sum_beta X[alpha][beta] * E[beta][col]  mod p(col),
// col = (comp, limb, j) over both ciphertext components and all RNS limbs.
// It is computed EXACTLY with 8-bit slices: X = sum_i x_i 2^(8i) (S_x slices),
// E = sum_j e_j 2^(8j) (4 slices of a 31-bit residue), and
//     acc_s = sum_{i+j=s} sum_beta x_i[alpha][beta] e_j[beta][col]
// accumulated in int32 TMEM by tcgen05.mma kind::i8 (u8 x u8 -> s32); the
// epilogue recombines v = sum_s acc_s 2^(8s) in 64-bit (terms s >= 4 folded as
// acc_s * (2^(8s) mod p)) and Barrett-reduces it.  Bounds (host-checked):
// acc_s < 4 * m * 255^2 < 2^31 for m <= 8192.
//
// CTA = one 128-row x 64-column output tile.  Warp roles: warp 0 lane 0 feeds
// a STAGES-deep ring of shared-memory stages with 1-D bulk async copies (the
// operands are stored pre-swizzled, so one copy per operand per k-block);
// warp 1 lane 0 issues S_x*4 MMAs per 32-byte k-step into S_x+3 accumulators;
// warps 4-7 drain TMEM (tcgen05.ld) and write C.
#include "internal.h"

namespace nimbus {

template <int SX>
struct TcCfg {
    static constexpr uint32_t BM = kBM, BN = kBNT, BK = kBK;
    static constexpr uint32_t A_BYTES = SX * BM * BK;
    static constexpr uint32_t B_BYTES = kSW * BN * BK;
    static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
    static constexpr uint32_t STAGES = (SX == 4) ? 2 : 3;
    static constexpr uint32_t NACC = SX + kSW - 1;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 256;
    static_assert(NACC * BN <= TMEM_COLS, "accumulators exceed TMEM");
};

template <int SX>
__global__ void __launch_bounds__(256, 1) k_cop_tc(Rns R, const uint8_t* __restrict__ Xt,
                                                   const uint8_t* __restrict__ Et, uint32_t k, uint32_t KB,
                                                   uint32_t ncol, uint32_t* __restrict__ C) {
    using Cfg = TcCfg<SX>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t ct = blockIdx.x, mt = blockIdx.y;

    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(tfull, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer: bulk copies of pre-swizzled operand tiles
            const uint8_t* a_src = Xt + (size_t)mt * KB * Cfg::A_BYTES;
            const uint8_t* b_src = Et + (size_t)ct * KB * Cfg::B_BYTES;
            const uint64_t pol_a = policy_evict_last();    // X tile: re-read by every column tile
            const uint64_t pol_b = policy_evict_first();   // Enc(W): streamed once
            for (uint32_t kb = 0; kb < KB; kb++) {
                const uint32_t s = kb % Cfg::STAGES, ph = (kb / Cfg::STAGES) & 1;
                if (kb >= Cfg::STAGES) mbar_wait(&empty[s], ph ^ 1);
                uint8_t* sa = smem + s * Cfg::STAGE;
                mbar_arrive_expect_tx(&full[s], Cfg::STAGE);
                bulk_g2s(sa, a_src + (size_t)kb * Cfg::A_BYTES, Cfg::A_BYTES, &full[s], pol_a);
                bulk_g2s(sa + Cfg::A_BYTES, b_src + (size_t)kb * Cfg::B_BYTES, Cfg::B_BYTES, &full[s], pol_b);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            constexpr uint32_t idesc = idesc_i8(Cfg::BM, Cfg::BN);
            for (uint32_t kb = 0; kb < KB; kb++) {
                const uint32_t s = kb % Cfg::STAGES, ph = (kb / Cfg::STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a0 = smem_u32(smem + s * Cfg::STAGE);
                const uint32_t b0 = a0 + Cfg::A_BYTES;
#pragma unroll
                for (uint32_t kk = 0; kk < Cfg::BK / 32; kk++) {
#pragma unroll
                    for (uint32_t i = 0; i < (uint32_t)SX; i++) {
                        const uint64_t ad = sdesc_kmajor_sw128(a0 + i * Cfg::BM * Cfg::BK + kk * 32);
#pragma unroll
                        for (uint32_t j = 0; j < kSW; j++) {
                            const uint64_t bd = sdesc_kmajor_sw128(b0 + j * Cfg::BN * Cfg::BK + kk * 32);
                            const bool first = (i + j <= 3) ? (i == 0) : (j == 3);
                            const uint32_t accum = (kb | kk) != 0 || !first;
                            mma_i8_ss(tmem + (i + j) * Cfg::BN, ad, bd, idesc, accum);
                        }
                    }
                }
                mma_commit(&empty[s]);   // frees the smem stage when these MMAs retire
            }
            mma_commit(tfull);           // accumulators final
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> exact recombination -> mod p
        const uint32_t ew = warp - 4;
        const uint32_t row = mt * Cfg::BM + ew * 32 + lane;
        const uint32_t col0 = ct * Cfg::BN;
        const uint32_t limb = (col0 / R.N) % R.L, p = R.p[limb];
        const uint64_t mu = R.mu[limb];
        mbar_wait(tfull, 0);
        tc_fence_after();
        const uint32_t tbase = tmem + ((ew * 32) << 16);
#pragma unroll 1
        for (uint32_t cc = 0; cc < Cfg::BN / 16; cc++) {
            uint32_t v[Cfg::NACC][16];
#pragma unroll
            for (uint32_t s = 0; s < Cfg::NACC; s++) tmem_ld16(tbase + s * Cfg::BN + cc * 16, v[s]);
            tmem_ld_wait();
            uint32_t out[16];
#pragma unroll
            for (uint32_t u = 0; u < 16; u++) {
                uint64_t x = (uint64_t)v[0][u];
#pragma unroll
                for (uint32_t s = 1; s < Cfg::NACC && s < 4; s++) x += (uint64_t)v[s][u] << (8 * s);
#pragma unroll
                for (uint32_t s = 4; s < Cfg::NACC; s++) x += (uint64_t)v[s][u] * R.pow8[limb][s];
                out[u] = mod64(x, p, mu);
            }
            if (row < k) {
                uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * ncol + col0 + cc * 16);
#pragma unroll
                for (uint32_t q = 0; q < 4; q++)
                    dst[q] = make_uint4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tmem, Cfg::TMEM_COLS);
    }
}

template <int SX>
static cudaError_t launch_sx(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k, uint32_t* d_C,
                             cudaStream_t st) {
    using Cfg = TcCfg<SX>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_cop_tc<SX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    dim3 grid(ncol / Cfg::BN, (k + Cfg::BM - 1) / Cfg::BM);
    k_cop_tc<SX><<<grid, 256, Cfg::SMEM, st>>>(c->rns, d_Xt, w->d_Et, k, w->KB, ncol, d_C);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_cop_tcgen05(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k,
                               uint32_t* d_C, cudaStream_t st) {
    switch (sx_of(c->rns.ell)) {
        case 1: return launch_sx<1>(c, w, d_Xt, k, d_C, st);
        case 2: return launch_sx<2>(c, w, d_Xt, k, d_C, st);
        default: return launch_sx<4>(c, w, d_Xt, k, d_C, st);
    }
}

}  // namespace nimbus
