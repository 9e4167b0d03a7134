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
// Structure (persistent, warp-specialised, one CTA per SM):
//   warp 0      producer: 1-D bulk async copies of the pre-swizzled operand
//               tiles (X slices of the M tile, the 4 E planes of the N tile)
//               into a STAGES-deep shared-memory ring (mbarrier full/empty)
//   warp 1      MMA issuer: per 32-byte k-step, S_x MMAs of 128 x 4*BN x 32 --
//               the 4 E planes are stacked along N, so one MMA whose D starts
//               at TMEM column BN*i writes x_i*e_j into acc_{i+j} for all j
//   warp 2      TMEM allocator
//   warps 4-11  epilogue: tcgen05.ld -> exact recombination -> mod p -> C,
//               overlapped with the next tile's MMAs when the accumulators
//               fit twice in TMEM (ell <= 16)
// Tiles are walked M-fastest so concurrently running CTAs share the E tile in L2.
#include "internal.h"

namespace nimbus {

template <int SX>
struct TcCfg {
    static constexpr uint32_t BM = kBM, BN = kBNT, BK = kBK;
    static constexpr uint32_t A_BYTES = SX * BM * BK;          // 16 KB per X slice
    static constexpr uint32_t B_BYTES = kSW * BN * BK;         // 24 KB (4 planes x 48 rows)
    static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
    static constexpr uint32_t STAGES = (SX == 4) ? 2 : (SX == 2 ? 3 : 4);
    static constexpr uint32_t NACC = SX + kSW - 1;
    static constexpr uint32_t ACC_COLS = NACC * BN;            // one accumulator set
    static constexpr uint32_t ACC_BUFS = (2 * 256 >= 2 * ACC_COLS && ACC_COLS <= 256) ? 2 : 1;
    static constexpr uint32_t BUF_STRIDE = 256;                // TMEM column offset of buffer 1
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr uint32_t EPI_WARPS = 8;
    static constexpr uint32_t THREADS = 128 + 32 * EPI_WARPS;
    static constexpr uint32_t CHUNK = 8;                       // columns per tcgen05.ld
    static constexpr uint32_t NCHUNK = BN / CHUNK;             // 6
    static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 256;
    static_assert(ACC_COLS <= TMEM_COLS, "accumulators exceed TMEM");
    static_assert(SMEM <= 232448, "shared memory");
    static_assert(NCHUNK % 2 == 0, "epilogue split");
};

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(taddr));
}

#ifdef NIMBUS_TRACE
// Debug-only timeline (globaltimer ns) per CTA: [0] start, [1] setup done,
// [2] producer past the PDL wait, [3] end; tile ti: [4+4ti] MMA start,
// [5+4ti] last MMA issued, [6+4ti] epilogue sees accumulators, [7+4ti] epilogue done.
__device__ uint64_t* g_trace = nullptr;
__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
#define TRACE(slot) do { if (g_trace && (slot) < 64) g_trace[blockIdx.x * 64 + (slot)] = gtimer(); } while (0)
extern "C" int nimbus_trace_set(void* p) { return (int)cudaMemcpyToSymbol(g_trace, &p, sizeof(p)); }
#else
#define TRACE(slot) do { } while (0)
#endif

template <int SX, int CL>
__global__ void __launch_bounds__(TcCfg<SX>::THREADS, 1)
k_cop_tc(Rns R, const uint8_t* __restrict__ Xt, const uint8_t* __restrict__ Et, uint32_t k, uint32_t Mt,
         uint32_t CT, uint32_t KB, uint32_t ncol, uint32_t* __restrict__ C) {
    // CL = cluster size along the column-tile dimension.  With CL = 2 the two
    // CTAs of a cluster work on column tiles (2q, 2q+1) of the same M tile in
    // lockstep; each fetches half of every X-slice block and multicasts it into
    // both CTAs' shared memory, halving the L2->SM traffic of the A operand.
    using Cfg = TcCfg<SX>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CL > 1 ? cluster_ctarank() : 0;
    const uint32_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
    const uint32_t nunits = Mt * (CT / CL);
    if (threadIdx.x == 0) TRACE(0);

    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], CL); }
        for (uint32_t b = 0; b < 2; b++) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], Cfg::EPI_WARPS); }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    if (CL > 1) cluster_sync(); else __syncthreads();   // partner barriers initialised before any multicast
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) TRACE(1);
    pdl_trigger();   // let the pack kernel's CTAs get resident early (they wait on us)

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer
            const uint64_t pol_a = policy_evict_last();    // X slices: reused by every N tile
            const uint64_t pol_b = policy_evict_first();   // Enc(W): streamed
            constexpr uint32_t A_PART = Cfg::A_BYTES / CL;
            uint32_t it = 0;
            bool waited = false;
            for (uint32_t u = cid; u < nunits; u += ncl) {
                const uint32_t mt = u % Mt, ct = (u / Mt) * CL + rank;
                const uint8_t* a_src = Xt + (size_t)mt * KB * Cfg::A_BYTES;
                const uint8_t* b_src = Et + (size_t)ct * KB * Cfg::B_BYTES;
                for (uint32_t kb = 0; kb < KB; kb++, it++) {
                    const uint32_t s = it % Cfg::STAGES, ph = (it / Cfg::STAGES) & 1;
                    if (it >= Cfg::STAGES) mbar_wait(&empty[s], ph ^ 1);   // freed by all CL consumers
                    uint8_t* sa = smem + s * Cfg::STAGE;
                    mbar_arrive_expect_tx(&full[s], Cfg::STAGE);
                    // Enc(W) is immutable: fetch it before waiting on the X-slicing kernel
                    bulk_g2s(sa + Cfg::A_BYTES, b_src + (size_t)kb * Cfg::B_BYTES, Cfg::B_BYTES, &full[s], pol_b);
                    if (!waited) { pdl_wait(); waited = true; TRACE(2); }
                    const uint8_t* asrc = a_src + (size_t)kb * Cfg::A_BYTES + rank * A_PART;
                    if (CL > 1) bulk_g2s_mc(sa + rank * A_PART, asrc, A_PART, &full[s], (1u << CL) - 1, pol_a);
                    else bulk_g2s(sa, asrc, A_PART, &full[s], pol_a);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer
            constexpr uint32_t idesc_full = idesc_i8(Cfg::BM, kSW * Cfg::BN);        // N = 192
            constexpr uint32_t idesc_lo = idesc_i8(Cfg::BM, (kSW - 1) * Cfg::BN);    // N = 144
            constexpr uint32_t idesc_one = idesc_i8(Cfg::BM, Cfg::BN);               // N = 48
            uint32_t it = 0, ti = 0;
            for (uint32_t u = cid; u < nunits; u += ncl, ti++) {
                const uint32_t buf = Cfg::ACC_BUFS == 2 ? (ti & 1) : 0;
                const uint32_t use = Cfg::ACC_BUFS == 2 ? (ti >> 1) : ti;
                if (ti >= Cfg::ACC_BUFS) mbar_wait(&tempty[buf], (use & 1) ^ 1);
                TRACE(4 + 4 * ti);
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
                        for (uint32_t i = 0; i < (uint32_t)SX; i++) {
                            const uint64_t ad = sdesc_kmajor_sw128(a0 + i * Cfg::BM * Cfg::BK + kk * 32);
                            if ((kb | kk) != 0 || i == 0) {
                                mma_i8_ss(dacc + i * Cfg::BN, ad, bd, idesc_full, (kb | kk) != 0);
                            } else {
                                // first k-step, i >= 1: acc_i..acc_{i+2} exist, acc_{i+3} is new
                                mma_i8_ss(dacc + i * Cfg::BN, ad, bd, idesc_lo, 1u);
                                const uint64_t bd3 =
                                    sdesc_kmajor_sw128(b0 + (kSW - 1) * Cfg::BN * Cfg::BK + kk * 32);
                                mma_i8_ss(dacc + (i + kSW - 1) * Cfg::BN, ad, bd3, idesc_one, 0u);
                            }
                        }
                    }
                    // frees the stage (in every CTA of the cluster) when these MMAs retire
                    if (CL > 1) mma_commit_mc(&empty[s], (1u << CL) - 1);
                    else mma_commit(&empty[s]);
                }
                mma_commit(&tfull[buf]);       // accumulator set complete
                TRACE(5 + 4 * ti);
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue
        const uint32_t ew = warp - 4;
        const uint32_t sub = ew & 3, half = ew >> 2;        // TMEM lane group, column half
        uint32_t ti = 0;
        for (uint32_t u = cid; u < nunits; u += ncl, ti++) {
            const uint32_t mt = u % Mt, ct = (u / Mt) * CL + rank;
            const uint32_t buf = Cfg::ACC_BUFS == 2 ? (ti & 1) : 0;
            const uint32_t use = Cfg::ACC_BUFS == 2 ? (ti >> 1) : ti;
            mbar_wait(&tfull[buf], use & 1);
            if (ew == 0 && lane == 0) TRACE(6 + 4 * ti);
            tc_fence_after();
            const uint32_t row = mt * Cfg::BM + sub * 32 + lane;
            const uint32_t tbase = tmem + ((sub * 32) << 16) + buf * Cfg::BUF_STRIDE;
            // Each warp drains CPW chunks of 8 columns for its 32 rows; BATCH chunks of
            // tcgen05.ld are issued before one wait (all of them when they fit in registers).
            constexpr uint32_t CPW = Cfg::NCHUNK / 2;
            constexpr uint32_t BATCH = (Cfg::NACC * 8 * CPW <= 128) ? CPW : 1;
#pragma unroll 1
            for (uint32_t c0 = 0; c0 < CPW; c0 += BATCH) {
                uint32_t v[BATCH][Cfg::NACC][8];
#pragma unroll
                for (uint32_t b = 0; b < BATCH; b++)
#pragma unroll
                    for (uint32_t s = 0; s < Cfg::NACC; s++)
                        tmem_ld8(tbase + s * Cfg::BN + (half * CPW + c0 + b) * Cfg::CHUNK, v[b][s]);
                tmem_ld_wait();
#pragma unroll
                for (uint32_t b = 0; b < BATCH; b++) {
                    const uint32_t col0 = ct * Cfg::BN + (half * CPW + c0 + b) * Cfg::CHUNK;
                    if (col0 >= ncol || row >= k) continue;
                    const uint32_t limb = (col0 / R.N) % R.L;
                    const uint32_t p = R.p[limb], c32 = R.c32[limb];
                    uint32_t out[8];
#ifdef NIMBUS_NOMATH
#pragma unroll
                    for (uint32_t u = 0; u < 8; u++) {
                        uint32_t x = 0;
#pragma unroll
                        for (uint32_t s = 0; s < Cfg::NACC; s++) x ^= v[b][s][u];
                        out[u] = x;
                    }
#else
#pragma unroll
                    for (uint32_t u = 0; u < 8; u++) {
                        // v = sum_s acc_s 2^(8s): s < 4 exact, s >= 4 as acc_s (2^(8s) mod p)  (< 2^64)
                        uint64_t x = mad_wide(v[b][1][u], 1u << 8, v[b][0][u]);
                        x = mad_wide(v[b][2][u], 1u << 16, x);
                        x = mad_wide(v[b][3][u], 1u << 24, x);
#pragma unroll
                        for (uint32_t s = 4; s < Cfg::NACC; s++) x = mad_wide(v[b][s][u], R.pow8[limb][s], x);
                        out[u] = reduce64_pm(x, p, c32);
                    }
#endif
#ifdef NIMBUS_NOSTORE
                    if (out[0] == 0x12345678u && out[7] == 0x9abcdef0u)
#endif
                    {
                        uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * ncol + col0);
                        dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
                        dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
            if (ew == 0 && lane == 0) TRACE(7 + 4 * ti);
        }
    }
    tc_fence_before();
    if (CL > 1) cluster_sync(); else __syncthreads();   // no CTA leaves while its partner may still signal it
    if (threadIdx.x == 0) TRACE(3);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, Cfg::TMEM_COLS);
    }
}

template <int SX, int CL>
static cudaError_t launch_sx(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k, uint32_t* d_C,
                             cudaStream_t st) {
    using Cfg = TcCfg<SX>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_cop_tc<SX, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)Cfg::SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    const uint32_t CT = col_tiles(c), Mt = (k + kBM - 1) / kBM;
    const uint32_t nunits = Mt * (CT / CL);
    uint32_t nclusters = (uint32_t)c->num_sms / CL;
    if (nunits < nclusters) nclusters = nunits;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nclusters * CL);
    cfg.blockDim = dim3(Cfg::THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CL;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cop_tc<SX, CL>, c->rns, d_Xt, (const uint8_t*)w->d_Et, k, Mt, CT,
                                       w->KB, ncol, d_C);
    c->launches++;
    return e;
}

cudaError_t launch_cop_tcgen05(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k,
                               uint32_t* d_C, cudaStream_t st) {
    switch (sx_of(c->rns.ell)) {
        case 1: return c->cluster == 2 ? launch_sx<1, 2>(c, w, d_Xt, k, d_C, st) : launch_sx<1, 1>(c, w, d_Xt, k, d_C, st);
        case 2: return c->cluster == 2 ? launch_sx<2, 2>(c, w, d_Xt, k, d_C, st) : launch_sx<2, 1>(c, w, d_Xt, k, d_C, st);
        default: return c->cluster == 2 ? launch_sx<4, 2>(c, w, d_Xt, k, d_C, st) : launch_sx<4, 1>(c, w, d_Xt, k, d_C, st);
    }
}

}  // namespace nimbus
