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
// acc_s * (2^(8s) mod p)) and reduces it mod p.  Bounds (host-checked):
// acc_s < 4 * m * 255^2 < 2^31 for m <= 8192.
//
// The 4 byte planes of an Enc(W) tile are stacked along N in shared memory
// (plane j = rows [BN j, BN j + BN)), so ONE MMA of N = 4 BN whose D starts at
// TMEM column BN*i writes x_i*e_j into acc_{i+j} for all four j at once.
//
// Two kernels, both persistent and warp-specialised (one CTA per SM):
//  k_cop_tc      streaming: every k-block brings its X slices and its E planes
//                through a shared-memory ring (bulk async copies).
//  k_cop_tc_res  resident X (ell <= 16, one 128-row M tile, m <= 768): the X
//                slices are fetched once per CTA -- slice 0 into TMEM (read by
//                the MMA as its A operand), slice 1 kept in shared memory --
//                and only Enc(W) streams.  The L2->SM traffic per tile drops
//                from (X + E) to E, which is what bounds the k = 128 layers.
// Roles: warp 0 producer, warp 1 MMA issuer, warp 2 TMEM allocator, warps 4-11
// epilogue (tcgen05.ld -> recombination -> mod p -> C), double-buffered TMEM
// accumulators when two sets fit so the epilogue overlaps the next tile.
#include <cstdio>
#include "internal.h"

namespace nimbus {

// D[tmem] (+)= A[tmem] * B[smem], kind::i8
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
        :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// (mma_i8_ts_w: common.cuh)
__device__ __forceinline__ void tmem_cp_128x256b_w(uint32_t taddr, uint64_t sdesc) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}"
        :: "r"(taddr), "l"(sdesc) : "memory");
}
// smem (SWIZZLE_128B K-major, 128 rows x 32 B) -> TMEM 128 lanes x 8 columns
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" :: "r"(taddr), "l"(sdesc) : "memory");
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

// ------------------------------------------------------------------ epilogue
// The epilogue warp has its accumulators in registers: hand the TMEM set back to the MMA
// issuer before the recombination / reduction / stores (warp-converged; one arrive per warp),
// so the next tile's MMAs into this set overlap the epilogue's arithmetic.
__device__ __forceinline__ void acc_release(uint64_t* bar) {
    tc_fence_before();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}

// ------------------------------------------------------------------ epilogue
// Warp (sub, half) drains rows [32 sub, 32 sub + 32) and half of the BN
// columns of one accumulator set: CPW chunks of 8 columns, BATCH chunks of
// tcgen05.ld per wait.  tacc = TMEM address of acc_0 for lane 32 sub.
template <uint32_t NACC, uint32_t BN>
__device__ __forceinline__ void epilogue_tile(const Rns& R, uint32_t tacc, uint32_t half, uint32_t row, uint32_t k,
                                              uint32_t col_base, uint32_t ncol, uint32_t* __restrict__ C,
                                              uint64_t* rel = nullptr) {
    constexpr uint32_t CPW = BN / 8 / 2;
    constexpr uint32_t BATCH = (NACC * 8 * CPW <= 128) ? CPW : 1;
#pragma unroll 1
    for (uint32_t c0 = 0; c0 < CPW; c0 += BATCH) {
        uint32_t v[BATCH][NACC][8];
#pragma unroll
        for (uint32_t b = 0; b < BATCH; b++)
#pragma unroll
            for (uint32_t s = 0; s < NACC; s++) tmem_ld8(tacc + s * BN + (half * CPW + c0 + b) * 8, v[b][s]);
        tmem_ld_wait();
        if (rel && c0 + BATCH >= CPW) acc_release(rel);   // last load done: the MMA may reuse the set
#pragma unroll
        for (uint32_t b = 0; b < BATCH; b++) {
            const uint32_t col0 = col_base + (half * CPW + c0 + b) * 8;
            if (col0 >= ncol || row >= k) continue;
            const uint32_t limb = (col0 / R.N) % R.L;
            const uint32_t p = R.p[limb], c32 = R.c32[limb];
            uint32_t out[8];
#ifdef NIMBUS_NOMATH
#pragma unroll
            for (uint32_t u = 0; u < 8; u++) {
                uint32_t x = 0;
#pragma unroll
                for (uint32_t s = 0; s < NACC; s++) x ^= v[b][s][u];
                out[u] = x;
            }
#else
#pragma unroll
            for (uint32_t u = 0; u < 8; u++) {
                // v = sum_s acc_s 2^(8s): s < 4 exact, s >= 4 as acc_s (2^(8s) mod p)  (< 2^64)
                uint64_t x = v[b][0][u];
                if (NACC > 1) x = mad_wide(v[b][1][u], 1u << 8, x);
                if (NACC > 2) x = mad_wide(v[b][2][u], 1u << 16, x);
                if (NACC > 3) x = mad_wide(v[b][3][u], 1u << 24, x);
#pragma unroll
                for (uint32_t s = 4; s < NACC; s++) x = mad_wide(v[b][s][u], R.pow8[limb][s], x);
                out[u] = reduce64_pm(x, p, c32);
            }
#endif
#ifdef NIMBUS_RES_NOSTORE
            if (out[0] != 0xFFFFFFFFu) continue;     // diagnostic (wrong results): practically no C stores
#endif
            uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * ncol + col0);
            dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
            dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
        }
    }
}

// Epilogue of the alternating-base single set (TcCfg::SPLIT): accumulators [F0, F1) first (the
// ones the next tile overwrites), then the rest.  v = sum_s acc_s 2^(8s) is summed in the same
// 64-bit terms as epilogue_tile (s < 4 shifted exactly, s >= 4 as acc_s (2^(8s) mod p); the sum
// stays < 2^64 in any order), the first part kept as one uint64 per output.
template <uint32_t NACC, uint32_t BN, uint32_t F0, uint32_t F1>
__device__ __forceinline__ void epilogue_split(const Rns& R, uint32_t tacc, uint32_t half, uint32_t row, uint32_t k,
                                               uint32_t col_base, uint32_t ncol, uint32_t* __restrict__ C,
                                               uint64_t* rel_first, uint64_t* rel_all) {
    constexpr uint32_t CPW = BN / 8 / 2;
    uint64_t P[CPW][8];
    auto term = [&](uint32_t s, uint32_t v, uint32_t limb) -> uint64_t {
        return s < 4 ? (uint64_t)v << (8 * s) : (uint64_t)v * R.pow8[limb][s];
    };
    {
        uint32_t v[CPW][F1 - F0][8];
#pragma unroll
        for (uint32_t b = 0; b < CPW; b++)
#pragma unroll
            for (uint32_t s = F0; s < F1; s++) tmem_ld8(tacc + s * BN + (half * CPW + b) * 8, v[b][s - F0]);
        tmem_ld_wait();
        acc_release(rel_first);
#pragma unroll
        for (uint32_t b = 0; b < CPW; b++) {
            const uint32_t limb = ((col_base + (half * CPW + b) * 8) / R.N) % R.L;
#pragma unroll
            for (uint32_t u = 0; u < 8; u++) {
                uint64_t x = 0;
#pragma unroll
                for (uint32_t s = F0; s < F1; s++) x += term(s, v[b][s - F0][u], limb);
                P[b][u] = x;
            }
        }
    }
    uint32_t v[CPW][NACC - (F1 - F0)][8];
#pragma unroll
    for (uint32_t b = 0; b < CPW; b++) {
        uint32_t q = 0;
#pragma unroll
        for (uint32_t s = 0; s < NACC; s++)
            if (s < F0 || s >= F1) tmem_ld8(tacc + s * BN + (half * CPW + b) * 8, v[b][q++]);
    }
    tmem_ld_wait();
    acc_release(rel_all);
#pragma unroll
    for (uint32_t b = 0; b < CPW; b++) {
        const uint32_t col0 = col_base + (half * CPW + b) * 8;
        if (col0 >= ncol || row >= k) continue;
        const uint32_t limb = (col0 / R.N) % R.L;
        uint32_t out[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; u++) {
            uint64_t x = P[b][u];
            uint32_t q = 0;
#pragma unroll
            for (uint32_t s = 0; s < NACC; s++)
                if (s < F0 || s >= F1) x += term(s, v[b][q++][u], limb);
            out[u] = reduce64_pm(x, R.p[limb], R.c32[limb]);
        }
        uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * ncol + col0);
        dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
        dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
    }
}

// ------------------------------------------------------------------ R = 1 fused epilogue
// Output of an R = 1 layer (n > N/2, L = 2 -> L_out = 1): packing is the identity
// (c~[theta] = c[theta], PAPER.md:672-679 with one row), so the epilogue itself does
// the mod-switch c_0 <- (c_0 - [c_1]_centered) p_1^-1 mod p_0
// and the mask b -= Emb_{q'}(r), r = word(seed, 6, theta N + J) >> (64 - ell)
// (§8(c) #13) -- the arithmetic of pack_item (pack_dev.cuh) for one
// unwrapped row.  The CTA takes the limb-0 and the limb-1 tile of the same
// (component, J) range back to back; on the limb-0 tile the thread keeps its
// reduced residues in `hold`, on the limb-1 tile it combines and stores the output
// ciphertext (and R for component 0) -- no C round trip and no pack launch.
struct FuseOut {
    uint32_t* cts;      // [row][comp][N] (L_out = 1)
    uint32_t* Rout;     // [row][n], or null (R produced elsewhere)
    uint64_t key;       // prg_key(seed, 6)
    uint32_t n;
};

// The mask of 8 consecutive slots (row, J..J+7) of component 0: r = word(seed, 6, row N + J + 1 + u)
// >> (64 - ell) is stored to R (the slots J + u < n), and Emb_{q'}(r) mod p_0 is returned in emb.
__device__ __forceinline__ void fused_mask8(const Rns& R, const FuseOut& fo, uint32_t row, uint32_t J,
                                            uint32_t (&emb)[8]) {
    uint64_t z = fo.key + 0x9E3779B97F4A7C15ULL * ((uint64_t)row * R.N + J + 1);
    uint32_t rm[8];
#pragma unroll
    for (uint32_t u = 0; u < 8; u++, z += 0x9E3779B97F4A7C15ULL) {
        rm[u] = (uint32_t)(mix64(z) >> (64 - R.ell));
        emb[u] = emb_fast16(rm[u], (uint32_t)R.qout_mod_t, R.ell, R.p[0], R.t_inv[0], R.t_inv_sh[0]);
    }
    if (!fo.Rout) return;
    uint32_t* rdst = fo.Rout + (size_t)row * fo.n + J;
    if (fo.n % 4 == 0 && J + 8 <= fo.n) {          // 16-byte aligned: J % 8 == 0, n % 4 == 0
        reinterpret_cast<uint4*>(rdst)[0] = make_uint4(rm[0], rm[1], rm[2], rm[3]);
        reinterpret_cast<uint4*>(rdst)[1] = make_uint4(rm[4], rm[5], rm[6], rm[7]);
    } else {
#pragma unroll
        for (uint32_t u = 0; u < 8; u++)
            if (J + u < fo.n) rdst[u] = rm[u];
    }
}

// pre: the component-0 masks of this tile were computed (and R stored) ahead of time, while the
// epilogue warps waited for their first accumulators (fused_mask8 into pre); else computed here.
template <uint32_t NACC, uint32_t BN>
__device__ __forceinline__ void epilogue_fused(const Rns& R, uint32_t tacc, uint32_t half, uint32_t row, uint32_t k,
                                               uint32_t col_base, bool second, uint32_t (&hold)[BN / 16][8],
                                               const FuseOut& fo, uint64_t* rel, bool use_pre,
                                               const uint32_t (&pre)[BN / 16][8]) {
    constexpr uint32_t CPW = BN / 8 / 2;
    uint32_t v[CPW][NACC][8];
#pragma unroll
    for (uint32_t b = 0; b < CPW; b++)
#pragma unroll
        for (uint32_t s = 0; s < NACC; s++) tmem_ld8(tacc + s * BN + (half * CPW + b) * 8, v[b][s]);
    tmem_ld_wait();
    acc_release(rel);                                   // accumulators in registers: free the set
    if (row >= k) return;
    const uint32_t N = R.N, limb = second ? 1 : 0;
    const uint32_t p = R.p[limb], c32 = R.c32[limb];
#pragma unroll
    for (uint32_t b = 0; b < CPW; b++) {
        uint32_t res[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; u++) {
            uint64_t x = v[b][0][u];
            if (NACC > 1) x = mad_wide(v[b][1][u], 1u << 8, x);
            if (NACC > 2) x = mad_wide(v[b][2][u], 1u << 16, x);
            if (NACC > 3) x = mad_wide(v[b][3][u], 1u << 24, x);
#pragma unroll
            for (uint32_t s = 4; s < NACC; s++) x = mad_wide(v[b][s][u], R.pow8[limb][s], x);
            res[u] = reduce64_pm(x, p, c32);
        }
        if (!second) {
#pragma unroll
            for (uint32_t u = 0; u < 8; u++) hold[b][u] = res[u];
            continue;
        }
        const uint32_t col0 = col_base + (half * CPW + b) * 8;
        const uint32_t comp = col0 / (2 * N), J = col0 % N;
        const uint32_t p0 = R.p[0], p1 = R.p[1];
        uint32_t out[8], emb[8];
        if (comp == 0) {
            if (use_pre) {
#pragma unroll
                for (uint32_t u = 0; u < 8; u++) emb[u] = pre[b][u];
            } else {
                fused_mask8(R, fo, row, J, emb);
            }
        }
#pragma unroll
        for (uint32_t u = 0; u < 8; u++) {
            const uint32_t c = res[u];
            const bool neg = c > (p1 >> 1);                 // centered rho = c - p_1 < 0
            const uint32_t mag = neg ? p1 - c : c;
            const uint32_t d = neg ? addmod(hold[b][u], mag, p0) : submod(hold[b][u], mag, p0);
            uint32_t o = mulmod_shoup(d, R.inv_p[1][0], R.inv_p_sh[1][0], p0);
            if (comp == 0) o = submod(o, emb[u], p0);
            out[u] = o;
        }
        uint4* dst = reinterpret_cast<uint4*>(fo.cts + ((size_t)row * 2 + comp) * N + J);
        dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
        dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
    }
}

// The i-th column tile of this CTA: round-robin over the grid, or (FUSE) round-robin
// over (component, J-tile) pairs, each pair's limb-0 and limb-1 tiles back to back.
template <bool FUSE>
struct TileSeq {
    uint32_t count, NT;
    __device__ TileSeq(uint32_t CT, uint32_t N, uint32_t BN) : NT(N / BN) {
        const uint32_t units = FUSE ? CT / 2 : CT;
        const uint32_t mine = blockIdx.x < units ? (units - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
        count = FUSE ? 2 * mine : mine;
    }
    __device__ uint32_t at(uint32_t ti) const {
        if (!FUSE) return blockIdx.x + ti * gridDim.x;
        const uint32_t pair = blockIdx.x + (ti >> 1) * gridDim.x;
        return (pair / NT) * 2 * NT + (ti & 1) * NT + pair % NT;
    }
};

// ------------------------------------------------------------------ streaming kernel
template <int SX, int BN_>
struct TcCfg {
    static constexpr uint32_t BM = kBM, BN = BN_, BK = kBK;
    static constexpr uint32_t A_BYTES = SX * BM * BK;          // 16 KB per X slice
    static constexpr uint32_t B_BYTES = kSW * BN * BK;         // 4 planes x BN rows x 128 B
    static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
    static constexpr uint32_t STAGES = (220u * 1024u) / STAGE > 6 ? 6 : (220u * 1024u) / STAGE;
    static constexpr uint32_t NACC = SX + kSW - 1;
    static constexpr uint32_t ACC_COLS = NACC * BN;            // one accumulator set
    static constexpr uint32_t ACC_BUFS = ACC_COLS <= 256 ? 2 : 1;
    static constexpr uint32_t BUF_STRIDE = 256;                // TMEM column offset of buffer 1
    static constexpr uint32_t TMEM_COLS = 512;
    // One set does not fit twice (S_x = 4, BN = 48: 7 x 48 = 336 columns): consecutive tiles
    // alternate between TMEM bases 0 and B1 = 512 - ACC_COLS, whose sets overlap in
    // [B1, ACC_COLS).  The epilogue of a base-0 tile drains the accumulators in that overlap
    // first (acc_LO_A..), of a base-B1 tile its acc_0..HI_B-1, and releases them before the
    // rest: the next tile's MMAs then wait for half an epilogue instead of a whole one.
#ifdef NIMBUS_NO_SPLIT
    static constexpr bool SPLIT = false;
#else
    static constexpr bool SPLIT = ACC_BUFS == 1 && ACC_COLS < TMEM_COLS;
#endif
    static constexpr uint32_t B1 = TMEM_COLS - ACC_COLS;
    static constexpr uint32_t LO_A = B1 / BN;                              // base 0: acc_LO_A.. overlap
    static constexpr uint32_t HI_B = (ACC_COLS - B1 + BN - 1) / BN;        // base B1: acc_0..HI_B-1 overlap
    static constexpr uint32_t EPI_WARPS = 8;
    static constexpr uint32_t THREADS = 128 + 32 * EPI_WARPS;
    static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 256;
    static_assert(ACC_COLS <= TMEM_COLS, "accumulators exceed TMEM");
    static_assert(!SPLIT || (LO_A >= 1 && HI_B <= NACC - 1), "split: both phases non-empty");
    static_assert(SMEM <= 232448, "shared memory");
    static_assert((BN / 8) % 2 == 0, "epilogue split");
};

template <int SX, int CL, int BN_>
__global__ void __launch_bounds__(TcCfg<SX, BN_>::THREADS, 1)
k_cop_tc(Rns R, const uint8_t* __restrict__ Xt, const uint8_t* __restrict__ Et, uint32_t k, uint32_t Mt,
         uint32_t CT, uint32_t KB, uint32_t ncol, uint32_t* __restrict__ C) {
    // CL = cluster size along the column-tile dimension.  With CL = 2 the two
    // CTAs of a cluster work on column tiles (2q, 2q+1) of the same M tile in
    // lockstep; each fetches half of every X-slice block and multicasts it into
    // both CTAs' shared memory (halves the L2 reads of the A operand).
    using Cfg = TcCfg<SX, BN_>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* trel = tempty + 2;      // SPLIT: full release of a tile, by tile parity
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(trel + 2);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CL > 1 ? cluster_ctarank() : 0;
    const uint32_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
    const uint32_t nunits = Mt * (CT / CL);
    if (threadIdx.x == 0) TRACE(0);

    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], CL); }
        for (uint32_t b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1); mbar_init(&tempty[b], Cfg::EPI_WARPS); mbar_init(&trel[b], Cfg::EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    if (CL > 1) cluster_sync(); else __syncthreads();   // partner barriers initialised before any multicast
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) TRACE(1);
#ifndef NIMBUS_LATE_TRIGGER
    pdl_trigger();   // let the pack kernel CTAs get resident early (they wait on us)
#endif

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
        {   // the whole warp, converged: one elected lane issues (warp-uniform operands)
            // ---------------- MMA issuer
            constexpr uint32_t idesc_full = idesc_i8(Cfg::BM, kSW * Cfg::BN);        // N = 4 BN
            constexpr uint32_t idesc_lo = idesc_i8(Cfg::BM, (kSW - 1) * Cfg::BN);    // N = 3 BN
            constexpr uint32_t idesc_one = idesc_i8(Cfg::BM, Cfg::BN);               // N = BN
            uint32_t it = 0, ti = 0;
            for (uint32_t u = cid; u < nunits; u += ncl, ti++) {
                const uint32_t buf = Cfg::ACC_BUFS == 2 ? (ti & 1) : 0;
                const uint32_t use = Cfg::ACC_BUFS == 2 ? (ti >> 1) : ti;
                uint32_t dacc;
                if constexpr (Cfg::SPLIT) {
                    // tile ti at base (ti & 1) B1: the previous tile's overlapping accumulators drained
                    // (its first-part release on tempty[0]), and the tile before it (same base) drained
                    // completely (trel[ti & 1]: only tiles of this parity arrive there, so the barrier
                    // cannot run two phases ahead of this wait)
                    if (ti >= 1) mbar_wait(&tempty[0], (ti - 1) & 1);
                    if (ti >= 2) mbar_wait(&trel[ti & 1], ((ti - 2) >> 1) & 1);
                    dacc = tmem + (ti & 1) * Cfg::B1;
                } else {
                    if (ti >= Cfg::ACC_BUFS) mbar_wait(&tempty[buf], (use & 1) ^ 1);
                    dacc = tmem + buf * Cfg::BUF_STRIDE;
                }
                TRACE(4 + 4 * ti);
                tc_fence_after();
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
                                mma_i8_ss_w(dacc + i * Cfg::BN, ad, bd, idesc_full, (kb | kk) != 0);
                            } else {
                                // first k-step, i >= 1: acc_i..acc_{i+2} exist, acc_{i+3} is new
                                mma_i8_ss_w(dacc + i * Cfg::BN, ad, bd, idesc_lo, 1u);
                                const uint64_t bd3 =
                                    sdesc_kmajor_sw128(b0 + (kSW - 1) * Cfg::BN * Cfg::BK + kk * 32);
                                mma_i8_ss_w(dacc + (i + kSW - 1) * Cfg::BN, ad, bd3, idesc_one, 0u);
                            }
                        }
                    }
                    // frees the stage (in every CTA of the cluster) when these MMAs retire
                    if (CL > 1) mma_commit_mc_w(&empty[s], (1u << CL) - 1);
                    else mma_commit_w(&empty[s]);
                }
                mma_commit_w(&tfull[buf]);       // accumulator set complete
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
            if constexpr (Cfg::SPLIT) {
                const uint32_t tl = tmem + ((sub * 32) << 16) + (ti & 1) * Cfg::B1;
                const uint32_t row = mt * Cfg::BM + sub * 32 + lane;
                if ((ti & 1) == 0)
                    epilogue_split<Cfg::NACC, Cfg::BN, Cfg::LO_A, Cfg::NACC>(R, tl, half, row, k, ct * Cfg::BN, ncol, C,
                                                                           &tempty[0], &trel[0]);
                else
                    epilogue_split<Cfg::NACC, Cfg::BN, 0, Cfg::HI_B>(R, tl, half, row, k, ct * Cfg::BN, ncol, C,
                                                                   &tempty[0], &trel[1]);
            } else {
                epilogue_tile<Cfg::NACC, Cfg::BN>(R, tmem + ((sub * 32) << 16) + buf * Cfg::BUF_STRIDE, half,
                                                 mt * Cfg::BM + sub * 32 + lane, k, ct * Cfg::BN, ncol, C, &tempty[buf]);
            }
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

// ------------------------------------------------------------------ resident-X kernel
// Shared memory: slice 1 of X resident (96 KB) and four 32 KB slots.  In the first tile the
// slots hold Enc(W) k-block pairs (slots 0, 1) and slice 0 of X on its way to TMEM (slots 2, 3),
// so that both Enc(W) and X of the first two k-block pairs, and all of slice 1, are requested in
// ONE round trip (the first tile used to wait for three: slice 0 went through one 32 KB staging
// buffer, pair by pair).  From the second tile on all four slots carry Enc(W) (128 KB in flight).
struct ResCfg {
    static constexpr uint32_t BM = kBM, BN = kBNR, BK = kBK, SX = 2;
    static constexpr uint32_t SLICE = BM * BK;                 // one X slice, one k-block: 16 KB
    static constexpr uint32_t B_BYTES = kSW * BN * BK;         // Enc(W) per k-block: 16 KB
    static constexpr uint32_t KPS = 2;                         // k-blocks per slot: one 32 KB bulk copy
    static constexpr uint32_t SLOT = KPS * B_BYTES;
    static constexpr uint32_t NSLOT = 4;
    static constexpr uint32_t NACC = SX + kSW - 1;             // 5
    static constexpr uint32_t ACC_COLS = NACC * BN;            // 160
    static constexpr uint32_t A0_COLS = kResMaxKB * (BK / 4);  // slice 0 in TMEM: 32 columns per k-block
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr uint32_t EPI_WARPS = 8;
    static constexpr uint32_t THREADS = 128 + 32 * EPI_WARPS;
    // smem: slice 1 resident [KB][16 KB] | slots [4][32 KB] | barriers
    static constexpr uint32_t OFF_A1 = 0, OFF_S = kResMaxKB * SLICE;
    static constexpr uint32_t OFF_BAR = OFF_S + NSLOT * SLOT;
    static constexpr size_t SMEM = (size_t)OFF_BAR + 1024 + 256;
    static_assert(A0_COLS + 2 * ACC_COLS <= TMEM_COLS, "TMEM budget");
    static_assert(SMEM <= 232448, "shared memory");
    static_assert(KPS * SLICE == SLOT, "a slot holds one k-block pair of slice 0");
    static_assert((kResMaxKB + KPS - 1) / KPS <= 3, "the first tile has at most 3 k-block pairs");
};

// Slot of Enc(W) message `it` >= KP (second tile on): the slots in the order the first tile
// frees them (its pair kp uses Enc(W) slot kp & 1 and slice-0 slot 2 + (kp & 1)), 4 nibbles per KP.
__device__ __forceinline__ uint32_t res_slot(uint32_t it, uint32_t KP) {
    const uint32_t order = KP == 3 ? 0x0213u : KP == 2 ? 0x1302u : 0x0231u;
    return (order >> (4 * ((it - KP) & 3))) & 0xFu;
}

// Several matmuls that share X (Q, K, V of a layer) run as one launch: the
// column tiles of their Enc(W)s are one tile sequence (tile t = job t / CT, tile t % CT), so X is
// fetched once per CTA and the launch streams all of their Enc(W) bytes with one ramp and one tail.
template <bool FUSE>
__global__ void __launch_bounds__(ResCfg::THREADS, 1)
k_cop_tc_res(Rns R, const uint8_t* __restrict__ Xt, ResJobs jobs, uint32_t k, uint32_t CT,
             uint32_t KB, uint32_t ncol, FuseOut fo, ResPf pf) {
    using Cfg = ResCfg;
    const TileSeq<FUSE> tiles(FUSE ? CT : CT * jobs.nj, R.N, Cfg::BN);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
    uint64_t* empty = full + Cfg::NSLOT;
    uint64_t* tfull = empty + Cfg::NSLOT;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const uint32_t KP = (KB + Cfg::KPS - 1) / Cfg::KPS;
    auto slot_ptr = [&](uint32_t s) { return smem + Cfg::OFF_S + s * Cfg::SLOT; };

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) TRACE(0);
    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < Cfg::NSLOT; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (uint32_t b = 0; b < 2; b++) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], Cfg::EPI_WARPS); }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) TRACE(1);
#ifndef NIMBUS_LATE_TRIGGER
    pdl_trigger();
#endif

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer
            const uint64_t pol_a = policy_evict_last();
            const uint64_t pol_b = policy_evict_first();
            // every use of a slot is released by one commit of the MMA issuer on empty[slot]
            uint32_t par = 0, seen = 0;
            auto acquire = [&](uint32_t s) {
                const uint32_t bit = 1u << s;
                if (seen & bit) mbar_wait(&empty[s], ((par & bit) ? 1u : 0u) ^ 1u);
                par ^= bit;
                seen |= bit;
            };
            // first tile: pairs 0 and 1 -- Enc(W) (immutable: fetched before the PDL wait), slice 0 of
            // X into slots 2, 3, all of slice 1 into its resident place -- in one round trip
            const uint32_t t0 = tiles.at(0);
            const uint8_t* e0 = jobs.Et[t0 / CT] + (size_t)(t0 % CT) * KB * Cfg::B_BYTES;
            const uint32_t P0 = KP < 2 ? KP : 2;
#ifdef NIMBUS_RES_XODD
            const bool nox = blockIdx.x & 1;    // diagnostic (wrong results): odd CTAs skip X (half the L2 hot-line reads)
#else
            constexpr bool nox = false;
#endif
            for (uint32_t kp = 0; kp < P0; kp++) {
                const uint32_t kb0 = kp * Cfg::KPS, nkb = min(Cfg::KPS, KB - kb0);
                acquire(kp);
                acquire(2 + kp);
                mbar_arrive_expect_tx(&full[kp], nkb * Cfg::B_BYTES +
                                      (nox ? 0u : nkb * Cfg::SLICE + (kp == 0 ? KB * Cfg::SLICE : 0)));
                bulk_g2s(slot_ptr(kp), e0 + (size_t)kb0 * Cfg::B_BYTES, nkb * Cfg::B_BYTES, &full[kp], pol_b);
            }
            // own later tiles towards L2 while the kernels before this one finish (their tail and the
            // pack leave DRAM idle); tiles 0 .. pf.from - 1 were prefetched by the previous contraction
            for (uint32_t ti = pf.from; ti < pf.from + pf.self && ti < tiles.count; ti++) {
                const uint32_t tg = tiles.at(ti);
                const uint8_t* p = jobs.Et[tg / CT] + (size_t)(tg % CT) * KB * Cfg::B_BYTES;
                for (uint32_t off = 0; off < KB * Cfg::B_BYTES; off += Cfg::SLOT)
                    prefetch_l2_bulk(p + off, min(Cfg::SLOT, KB * Cfg::B_BYTES - off));
            }
            pdl_wait();
            TRACE(2);
            if (!nox)
            for (uint32_t kb = 0; kb < KB; kb++)        // Xt[0][kb][slice]
                bulk_g2s(smem + Cfg::OFF_A1 + kb * Cfg::SLICE, Xt + ((size_t)kb * 2 + 1) * Cfg::SLICE, Cfg::SLICE,
                         &full[0], pol_a);
            for (uint32_t kp = 0; kp < P0; kp++) {
                const uint32_t kb0 = kp * Cfg::KPS, nkb = min(Cfg::KPS, KB - kb0);
                if (!nox)
                for (uint32_t q = 0; q < nkb; q++)
                    bulk_g2s(slot_ptr(2 + kp) + q * Cfg::SLICE, Xt + (size_t)(kb0 + q) * 2 * Cfg::SLICE, Cfg::SLICE,
                             &full[kp], pol_a);
            }
            if (KP == 3) {                              // pair 2 reuses pair 0's slots
                const uint32_t kb0 = 2 * Cfg::KPS, nkb = KB - kb0;
                acquire(0);
                acquire(2);
                mbar_arrive_expect_tx(&full[0], nkb * (Cfg::B_BYTES + (nox ? 0u : Cfg::SLICE)));
                bulk_g2s(slot_ptr(0), e0 + (size_t)kb0 * Cfg::B_BYTES, nkb * Cfg::B_BYTES, &full[0], pol_b);
                if (!nox)
                for (uint32_t q = 0; q < nkb; q++)
                    bulk_g2s(slot_ptr(2) + q * Cfg::SLICE, Xt + (size_t)(kb0 + q) * 2 * Cfg::SLICE, Cfg::SLICE,
                             &full[0], pol_a);
            }
            // later tiles: Enc(W) only, through all four slots
            uint32_t it = KP;
            for (uint32_t ti = 1; ti < tiles.count; ti++) {
                const uint32_t tg = tiles.at(ti), ct = tg % CT;
                const uint8_t* b_src = jobs.Et[tg / CT] + (size_t)ct * KB * Cfg::B_BYTES;
                for (uint32_t kp = 0; kp < KP; kp++, it++) {
                    const uint32_t s = res_slot(it, KP);
                    const uint32_t kb0 = kp * Cfg::KPS, nkb = min(Cfg::KPS, KB - kb0);
                    acquire(s);
                    if (ti == 1 && kp < 8) TRACE(52 + kp);
                    mbar_arrive_expect_tx(&full[s], nkb * Cfg::B_BYTES);
                    bulk_g2s(slot_ptr(s), b_src + (size_t)kb0 * Cfg::B_BYTES, nkb * Cfg::B_BYTES, &full[s], pol_b);
                }
            }
            // all of this CTA's copies are issued: pull the tile that CTA blockIdx.x of the next
            // contraction starts with towards L2 (nimbus_cop_prefetch_next; a hint, no completion)
            if (pf.base != nullptr && blockIdx.x < pf.grid) {
                const uint32_t b = blockIdx.x;
                for (uint32_t ti = 0; ti < pf.count; ti++) {          // that CTA's tiles.at(ti)
                    const uint32_t pair = b + (ti >> 1) * pf.grid;
                    const uint32_t t = pf.fuse ? (pair / pf.NT) * 2 * pf.NT + (ti & 1) * pf.NT + pair % pf.NT
                                               : b + ti * pf.grid;
                    if (t >= pf.ntiles) break;
                    const uint8_t* p = pf.base + (size_t)t * pf.tile_bytes;
                    for (uint32_t off = 0; off < pf.tile_bytes; off += Cfg::SLOT) {
                        const uint32_t nb = min(Cfg::SLOT, pf.tile_bytes - off);
                        if (pf.pol == 1) prefetch_l2_bulk(p + off, nb, pol_a);                       // evict_last
                        else if (pf.pol == 2) prefetch_l2_bulk(p + off, nb, policy_evict_normal());
                        else prefetch_l2_bulk(p + off, nb);
                    }
                }
            }
        }
    } else if (warp == 1) {
        {   // the whole warp, converged: one elected lane issues (warp-uniform operands)
            // ---------------- MMA issuer
            constexpr uint32_t idesc_full = idesc_i8(Cfg::BM, kSW * Cfg::BN);        // N = 128
            constexpr uint32_t idesc_lo = idesc_i8(Cfg::BM, (kSW - 1) * Cfg::BN);    // N = 96
            constexpr uint32_t idesc_one = idesc_i8(Cfg::BM, Cfg::BN);               // N = 32
            uint32_t it = 0, fpar = 0;
            for (uint32_t ti = 0; ti < tiles.count; ti++) {
                const uint32_t buf = ti & 1, use = ti >> 1;
                if (ti >= 2) mbar_wait(&tempty[buf], (use & 1) ^ 1);
                TRACE(4 + 4 * ti);
                tc_fence_after();
                const uint32_t dacc = tmem + Cfg::A0_COLS + buf * Cfg::ACC_COLS;
                for (uint32_t kp = 0; kp < KP; kp++, it++) {
                    const uint32_t s = ti == 0 ? (kp & 1) : res_slot(it, KP), bit = 1u << s;
                    const uint32_t kb0 = kp * Cfg::KPS, nkb = min(Cfg::KPS, KB - kb0);
                    mbar_wait(&full[s], (fpar & bit) ? 1u : 0u);
                    fpar ^= bit;
                    if (ti == 1 && kp < 8) TRACE(40 + kp);
                    tc_fence_after();
                    if (ti == 0) {
                        // first tile: this pair's slice 0 -> TMEM (in issue order with the MMAs), then its slot is free
                        const uint32_t xs = 2 + (kp & 1);
                        for (uint32_t q = 0; q < nkb; q++) {
                            const uint32_t stg = smem_u32(slot_ptr(xs) + q * Cfg::SLICE);
#pragma unroll
                            for (uint32_t kk = 0; kk < Cfg::BK / 32; kk++)
                                tmem_cp_128x256b_w(tmem + (kb0 + q) * (Cfg::BK / 4) + kk * 8, sdesc_kmajor_sw128(stg + kk * 32));
                        }
                        mma_commit_w(&empty[xs]);
                    }
#ifdef NIMBUS_RES_NOMMA
                    if (ti > 0) { mma_commit_w(&empty[s]); continue; }   // diagnostic (wrong results): stream only
#endif
                    for (uint32_t q = 0; q < nkb; q++) {
                        const uint32_t kb = kb0 + q;
                        const uint32_t a0t = tmem + kb * (Cfg::BK / 4);                      // slice 0, TMEM
                        const uint32_t a1 = smem_u32(smem + Cfg::OFF_A1 + kb * Cfg::SLICE);  // slice 1, smem
                        const uint32_t b0 = smem_u32(slot_ptr(s) + q * Cfg::B_BYTES);
#pragma unroll
                        for (uint32_t kk = 0; kk < Cfg::BK / 32; kk++) {
                            const uint64_t bd = sdesc_kmajor_sw128(b0 + kk * 32);
                            const uint32_t first = (kb | kk) == 0;
                            mma_i8_ts_w(dacc, a0t + kk * 8, bd, idesc_full, !first);          // x_0 e_j -> acc_j
                            const uint64_t ad1 = sdesc_kmajor_sw128(a1 + kk * 32);
                            if (!first) {
                                mma_i8_ss_w(dacc + Cfg::BN, ad1, bd, idesc_full, 1u);          // x_1 e_j -> acc_{j+1}
                            } else {
                                mma_i8_ss_w(dacc + Cfg::BN, ad1, bd, idesc_lo, 1u);
                                const uint64_t bd3 = sdesc_kmajor_sw128(b0 + (kSW - 1) * Cfg::BN * Cfg::BK + kk * 32);
                                mma_i8_ss_w(dacc + kSW * Cfg::BN, ad1, bd3, idesc_one, 0u);
                            }
                        }
                    }
                    mma_commit_w(&empty[s]);
                }
                mma_commit_w(&tfull[buf]);
                TRACE(5 + 4 * ti);
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue
        const uint32_t ew = warp - 4;
        const uint32_t sub = ew & 3, half = ew >> 2;
        uint32_t hold[Cfg::BN / 16][8];
        // FUSE: the masks of the CTA's first component-0 output tile (a limb-1 tile, odd ti) are
        // computed before its first accumulators are ready (the epilogue warps are idle then), and
        // its R stored once the previous grid is done (pdl_wait: R may be its output too)
        uint32_t pre[Cfg::BN / 16][8];
        uint32_t pre_ti = ~0u;
        if (FUSE) {
            for (uint32_t ti = 1; ti < tiles.count; ti += 2)
                if ((tiles.at(ti) % CT) * Cfg::BN < 2 * R.N) { pre_ti = ti; break; }
            const uint32_t row = sub * 32 + lane;
            if (pre_ti != ~0u && row < k) {
                pdl_wait();
                const uint32_t col_base = (tiles.at(pre_ti) % CT) * Cfg::BN;
#pragma unroll
                for (uint32_t b = 0; b < Cfg::BN / 16; b++)
                    fused_mask8(R, fo, row, (col_base + (half * (Cfg::BN / 16) + b) * 8) % R.N, pre[b]);
            }
        }
        for (uint32_t ti = 0; ti < tiles.count; ti++) {
            const uint32_t tg = tiles.at(ti), ct = tg % CT;
            const uint32_t buf = ti & 1, use = ti >> 1;
            mbar_wait(&tfull[buf], use & 1);
            if (ew == 0 && lane == 0) TRACE(6 + 4 * ti);
            tc_fence_after();
#ifdef NIMBUS_RES_NOEPI
            acc_release(&tempty[buf]);
            if (false)        // diagnostic (wrong results): no epilogue work at all
#endif
            if (FUSE)
                epilogue_fused<Cfg::NACC, Cfg::BN>(R, tmem + ((sub * 32) << 16) + Cfg::A0_COLS + buf * Cfg::ACC_COLS,
                                                   half, sub * 32 + lane, k, ct * Cfg::BN, ti & 1, hold, fo, &tempty[buf],
                                                   ti == pre_ti, pre);
            else
                epilogue_tile<Cfg::NACC, Cfg::BN>(R, tmem + ((sub * 32) << 16) + Cfg::A0_COLS + buf * Cfg::ACC_COLS,
                                                  half, sub * 32 + lane, k, ct * Cfg::BN, ncol, jobs.C[tg / CT],
                                                  &tempty[buf]);
            if (ew == 0 && lane == 0) TRACE(7 + 4 * ti);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TRACE(3);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, Cfg::TMEM_COLS);
    }
}

// ------------------------------------------------------------------ resident-X kernel, deep E ring
// Same contraction as k_cop_tc_res, with the shared memory given to the Enc(W)
// stream instead: slice 0 (all k-blocks) AND slice 1 of k-blocks 0..3 live in
// TMEM (both read by `kind::i8` MMAs as A from TMEM), only slice 1 of k-blocks
// 4..5 stays in shared memory, and one accumulator set (5 x 32 columns) is
// released by the epilogue as soon as it has been loaded into registers (the
// recombination and the stores then overlap the next tile's MMAs).  TMEM:
// 192 + 128 + 160 = 480 columns.  Shared memory: 32 KB of slice 1 + a 6-slot
// ring of 32 KB (192 KB; k_cop_tc_res: 96 KB).  Why: at k = 128 the MMAs of a
// 32 KB slot (~0.53 us) hold it out of the stream, so with 3 slots only ~2 are
// in flight and the per-SM Enc(W) rate stays at ~30 GB/s; a short cold stream
// needs more bytes in flight per SM than that (tools/stream_prefetch.cu).
// Ring messages, in the order producer and MMA issuer both follow: every
// (tile, k-block pair) kp is one E message; in the first tile it is followed by
// an X0 message (slice 0 of the pair -> TMEM) and, for pairs below k-block 4, an
// X1 message (slice 1 -> TMEM); slice 1 of pairs from k-block 4 on is copied
// straight into its resident place on the X0 message's barrier.
struct ResCfg2 {
    static constexpr uint32_t BM = kBM, BN = kBNR, BK = kBK, SX = 2;
    static constexpr uint32_t SLICE = BM * BK;                 // one X slice, one k-block: 16 KB
    static constexpr uint32_t B_BYTES = kSW * BN * BK;         // Enc(W) per k-block: 16 KB
    static constexpr uint32_t KPS = 2;                         // k-blocks per message: 32 KB
    static constexpr uint32_t SLOT = KPS * B_BYTES;
    static constexpr uint32_t STAGES = 6;
    static constexpr uint32_t T1 = 4;                          // slice-1 k-blocks in TMEM
    static constexpr uint32_t NACC = SX + kSW - 1;             // 5
    static constexpr uint32_t ACC_COLS = NACC * BN;            // 160
    static constexpr uint32_t A0_COL = 0, A1_COL = kResMaxKB * (BK / 4), ACC_COL = A1_COL + T1 * (BK / 4);
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr uint32_t EPI_WARPS = 8;
    static constexpr uint32_t THREADS = 128 + 32 * EPI_WARPS;
    // smem: slice 1 k-blocks T1.. [KB - T1][16 KB] | ring [STAGES][32 KB]
    static constexpr uint32_t OFF_A1 = 0, OFF_B = (kResMaxKB - T1) * SLICE;
    static constexpr size_t SMEM = (size_t)OFF_B + STAGES * SLOT + 1024 + 256;
    static_assert(ACC_COL + ACC_COLS <= TMEM_COLS, "TMEM budget");
    static_assert(SMEM <= 232448, "shared memory");
    static_assert(T1 % KPS == 0, "a k-block pair is either in TMEM or in smem");
    static_assert(SLOT == KPS * SLICE, "an X message fills one slot");
};

__global__ void __launch_bounds__(ResCfg2::THREADS, 1)
k_cop_tc_res2(Rns R, const uint8_t* __restrict__ Xt, const uint8_t* __restrict__ Et, uint32_t k, uint32_t CT,
              uint32_t KB, uint32_t ncol, uint32_t* __restrict__ C) {
    using Cfg = ResCfg2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_B + Cfg::STAGES * Cfg::SLOT);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) TRACE(0);
    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(tfull, 1);
        mbar_init(tempty, Cfg::EPI_WARPS);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) TRACE(1);
    pdl_trigger();
    const uint32_t KP = (KB + Cfg::KPS - 1) / Cfg::KPS;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer
            const uint64_t pol_a = policy_evict_last();
            const uint64_t pol_b = policy_evict_first();
            uint32_t it = 0, ti = 0;
            auto acquire = [&](uint32_t bytes) {
                const uint32_t s = it % Cfg::STAGES;
                if (it >= Cfg::STAGES) mbar_wait(&empty[s], ((it / Cfg::STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], bytes);
                it++;
                return s;
            };
            for (uint32_t ct = blockIdx.x; ct < CT; ct += gridDim.x, ti++) {
                const uint8_t* b_src = Et + (size_t)ct * KB * Cfg::B_BYTES;
                for (uint32_t kp = 0; kp < KP; kp++) {
                    const uint32_t kb0 = kp * Cfg::KPS, nkb = min(Cfg::KPS, KB - kb0);
                    uint32_t s = acquire(nkb * Cfg::B_BYTES);
                    bulk_g2s(smem + Cfg::OFF_B + s * Cfg::SLOT, b_src + (size_t)kb0 * Cfg::B_BYTES,
                             nkb * Cfg::B_BYTES, &full[s], pol_b);
                    if (ti == 0) {
                        if (kp == 0) { pdl_wait(); TRACE(2); }
                        const bool res1 = kb0 >= Cfg::T1;          // slice 1 of this pair resident in smem
                        s = acquire(nkb * Cfg::SLICE * (res1 ? 2 : 1));
                        for (uint32_t q = 0; q < nkb; q++) {
                            const uint8_t* xsrc = Xt + (size_t)(kb0 + q) * 2 * Cfg::SLICE;   // Xt[kb][slice]
                            bulk_g2s(smem + Cfg::OFF_B + s * Cfg::SLOT + q * Cfg::SLICE, xsrc, Cfg::SLICE, &full[s],
                                     pol_a);
                            if (res1)
                                bulk_g2s(smem + Cfg::OFF_A1 + (kb0 + q - Cfg::T1) * Cfg::SLICE, xsrc + Cfg::SLICE,
                                         Cfg::SLICE, &full[s], pol_a);
                        }
                        if (!res1) {
                            s = acquire(nkb * Cfg::SLICE);
                            for (uint32_t q = 0; q < nkb; q++)
                                bulk_g2s(smem + Cfg::OFF_B + s * Cfg::SLOT + q * Cfg::SLICE,
                                         Xt + (size_t)(kb0 + q) * 2 * Cfg::SLICE + Cfg::SLICE, Cfg::SLICE, &full[s],
                                         pol_a);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        {   // the whole warp, converged: one elected lane issues (warp-uniform operands)
            // ---------------- MMA issuer
            constexpr uint32_t idesc_full = idesc_i8(Cfg::BM, kSW * Cfg::BN);        // N = 128
            constexpr uint32_t idesc_lo = idesc_i8(Cfg::BM, (kSW - 1) * Cfg::BN);    // N = 96
            constexpr uint32_t idesc_one = idesc_i8(Cfg::BM, Cfg::BN);               // N = 32
            const uint32_t dacc = tmem + Cfg::ACC_COL;
            uint32_t it = 0, ti = 0;
            auto take = [&]() {
                const uint32_t s = it % Cfg::STAGES;
                mbar_wait(&full[s], (it / Cfg::STAGES) & 1);
                it++;
                tc_fence_after();
                return s;
            };
            // X message in slot s: k-blocks kb0.. of one slice -> TMEM columns col0 + 32 kb
            auto x_to_tmem = [&](uint32_t s, uint32_t kb0, uint32_t nkb, uint32_t col0) {
                for (uint32_t q = 0; q < nkb; q++) {
                    const uint32_t stg = smem_u32(smem + Cfg::OFF_B + s * Cfg::SLOT + q * Cfg::SLICE);
#pragma unroll
                    for (uint32_t kk = 0; kk < Cfg::BK / 32; kk++)
                        tmem_cp_128x256b_w(tmem + col0 + (kb0 + q) * (Cfg::BK / 4) + kk * 8,
                                         sdesc_kmajor_sw128(stg + kk * 32));
                }
                mma_commit_w(&empty[s]);
            };
            for (uint32_t ct = blockIdx.x; ct < CT; ct += gridDim.x, ti++) {
                if (ti >= 1) mbar_wait(tempty, (ti - 1) & 1);     // previous tile's accumulators are in registers
                TRACE(4 + 4 * ti);
                tc_fence_after();
                for (uint32_t kp = 0; kp < KP; kp++) {
                    const uint32_t kb0 = kp * Cfg::KPS, nkb = min(Cfg::KPS, KB - kb0);
                    const uint32_t sE = take();
                    if (ti == 0) {
                        x_to_tmem(take(), kb0, nkb, Cfg::A0_COL);
                        if (kb0 < Cfg::T1) x_to_tmem(take(), kb0, nkb, Cfg::A1_COL);
                    }
                    for (uint32_t q = 0; q < nkb; q++) {
                        const uint32_t kb = kb0 + q;
                        const uint32_t b0 = smem_u32(smem + Cfg::OFF_B + sE * Cfg::SLOT + q * Cfg::B_BYTES);
                        const bool t1 = kb < Cfg::T1;
                        const uint32_t a1s = t1 ? 0u : smem_u32(smem + Cfg::OFF_A1 + (kb - Cfg::T1) * Cfg::SLICE);
#pragma unroll
                        for (uint32_t kk = 0; kk < Cfg::BK / 32; kk++) {
                            const uint64_t bd = sdesc_kmajor_sw128(b0 + kk * 32);
                            const uint32_t first = (kb | kk) == 0;
                            mma_i8_ts_w(dacc, tmem + Cfg::A0_COL + kb * (Cfg::BK / 4) + kk * 8, bd, idesc_full, !first);
                            const uint32_t a1t = tmem + Cfg::A1_COL + kb * (Cfg::BK / 4) + kk * 8;
                            if (!first) {
                                if (t1) mma_i8_ts_w(dacc + Cfg::BN, a1t, bd, idesc_full, 1u);
                                else mma_i8_ss_w(dacc + Cfg::BN, sdesc_kmajor_sw128(a1s + kk * 32), bd, idesc_full, 1u);
                            } else {
                                // acc_1..3 accumulate onto x_0's first products, acc_4 starts here (kb 0 is in TMEM)
                                const uint64_t bd3 = sdesc_kmajor_sw128(b0 + (kSW - 1) * Cfg::BN * Cfg::BK + kk * 32);
                                mma_i8_ts_w(dacc + Cfg::BN, a1t, bd, idesc_lo, 1u);
                                mma_i8_ts_w(dacc + kSW * Cfg::BN, a1t, bd3, idesc_one, 0u);
                            }
                        }
                    }
                    mma_commit_w(&empty[sE]);
                }
                mma_commit_w(tfull);
                TRACE(5 + 4 * ti);
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: load the whole set, release it, then recombine and store
        const uint32_t ew = warp - 4;
        const uint32_t sub = ew & 3, half = ew >> 2;
        const uint32_t row = sub * 32 + lane;
        constexpr uint32_t CPW = Cfg::BN / 8 / 2;                 // 2 chunks of 8 columns per warp
        const uint32_t tacc = tmem + ((sub * 32) << 16) + Cfg::ACC_COL;
        uint32_t ti = 0;
        for (uint32_t ct = blockIdx.x; ct < CT; ct += gridDim.x, ti++) {
            mbar_wait(tfull, ti & 1);
            if (ew == 0 && lane == 0) TRACE(6 + 4 * ti);
            tc_fence_after();
            uint32_t v[CPW][Cfg::NACC][8];
#pragma unroll
            for (uint32_t b = 0; b < CPW; b++)
#pragma unroll
                for (uint32_t s = 0; s < Cfg::NACC; s++) tmem_ld8(tacc + s * Cfg::BN + (half * CPW + b) * 8, v[b][s]);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
#pragma unroll
            for (uint32_t b = 0; b < CPW; b++) {
                const uint32_t col0 = ct * Cfg::BN + (half * CPW + b) * 8;
                if (col0 >= ncol || row >= k) continue;
                const uint32_t limb = (col0 / R.N) % R.L;
                const uint32_t p = R.p[limb], c32 = R.c32[limb];
                uint32_t out[8];
#pragma unroll
                for (uint32_t u = 0; u < 8; u++) {
                    uint64_t x = v[b][0][u];
                    x = mad_wide(v[b][1][u], 1u << 8, x);
                    x = mad_wide(v[b][2][u], 1u << 16, x);
                    x = mad_wide(v[b][3][u], 1u << 24, x);
                    x = mad_wide(v[b][4][u], R.pow8[limb][4], x);
                    out[u] = reduce64_pm(x, p, c32);
                }
                uint4* dst = reinterpret_cast<uint4*>(C + (size_t)row * ncol + col0);
                dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
                dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
            }
            if (ew == 0 && lane == 0) TRACE(7 + 4 * ti);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TRACE(3);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, Cfg::TMEM_COLS);
    }
}

// ------------------------------------------------------------------ transposed kernel (ell = 32)
// D[coefficient column][row]: the 4 Enc(W) byte planes are the MMA A operand
// (M = 128 coefficient columns per plane) and the 4 X slices of a 64-row tile
// are stacked along N = 256, so one MMA per (plane j, 32-byte k-step) with D at
// TMEM column 64 j writes x_i e_j into acc_{i+j} (columns [64(i+j), +64)).  Per
// k-block it moves 64 KB of E + 32 KB of X into shared memory for 8192
// outputs, against 64 KB of X + 24 KB of E for 6144 in the streaming kernel:
// the L2->SM delivery rate is what bounds ell = 32.  The epilogue thread owns
// one coefficient column and writes rows, so stores are coalesced across lanes.
// RT_ X rows per tile: 256 / S_x fills N = 256 (one accumulator set: 7 x 64 or
// 11 x 32 TMEM columns); RT_ = 32 at S_x = 4 (N = 128, 7 x 32 = 224 columns) leaves
// room for two accumulator sets, so the epilogue of one tile overlaps the MMAs of
// the next -- with one set, the short m = 768 matmuls of C5 (6 k-blocks a tile)
// idle the tensor pipe for every epilogue -- at the price of more shared-memory
// fill per MAC (80 KB per 1024 MMA cycles instead of 96 KB per 2048).
// Transposed-kernel epilogue of the alternating-base single set (TCfgT::SPLIT): lane = one
// coefficient column, CH chunks of 8 rows; accumulators [F0, F1) of every chunk first (released),
// then the rest; the same 64-bit terms as the single-set epilogue, the first part kept per row.
template <uint32_t NACC, uint32_t RT, uint32_t CH, uint32_t F0, uint32_t F1>
__device__ __forceinline__ void epilogue_t_split(const Rns& R, uint32_t tb, uint32_t row0, uint32_t col, uint32_t limb,
                                                 uint32_t k, uint32_t ncol, uint32_t* __restrict__ C,
                                                 uint64_t* rel_first, uint64_t* rel_all) {
    auto term = [&](uint32_t s, uint32_t v) -> uint64_t {
        return s < 4 ? (uint64_t)v << (8 * s) : (uint64_t)v * R.pow8[limb][s];
    };
    uint64_t P[CH][8];
    {
        uint32_t v[CH][F1 - F0][8];
#pragma unroll
        for (uint32_t c = 0; c < CH; c++)
#pragma unroll
            for (uint32_t s = F0; s < F1; s++) tmem_ld8(tb + s * RT + c * 8, v[c][s - F0]);
        tmem_ld_wait();
        acc_release(rel_first);
#pragma unroll
        for (uint32_t c = 0; c < CH; c++)
#pragma unroll
            for (uint32_t q = 0; q < 8; q++) {
                uint64_t x = 0;
#pragma unroll
                for (uint32_t s = F0; s < F1; s++) x += term(s, v[c][s - F0][q]);
                P[c][q] = x;
            }
    }
    uint32_t v[CH][NACC - (F1 - F0)][8];
#pragma unroll
    for (uint32_t c = 0; c < CH; c++) {
        uint32_t i = 0;
#pragma unroll
        for (uint32_t s = 0; s < NACC; s++)
            if (s < F0 || s >= F1) tmem_ld8(tb + s * RT + c * 8, v[c][i++]);
    }
    tmem_ld_wait();
    acc_release(rel_all);
    const uint32_t p = R.p[limb], c32 = R.c32[limb];
#pragma unroll
    for (uint32_t c = 0; c < CH; c++)
#pragma unroll
        for (uint32_t q = 0; q < 8; q++) {
            uint64_t x = P[c][q];
            uint32_t i = 0;
#pragma unroll
            for (uint32_t s = 0; s < NACC; s++)
                if (s < F0 || s >= F1) x += term(s, v[c][i++][q]);
            const uint32_t row = row0 + c * 8 + q;
            if (row < k && col < ncol) C[(size_t)row * ncol + col] = reduce64_pm(x, p, c32);
        }
}

template <int SX_, int RT_ = 256 / SX_>
struct TCfgT {
    static constexpr uint32_t BM = kBNW, RT = RT_, BK = kBK, SX = SX_;
    static constexpr uint32_t A_BYTES = kSW * BM * BK;     // 64 KB: 4 planes x 128 columns x 128 B
    static constexpr uint32_t B_BYTES = SX * RT * BK;      // S_x slices x RT rows x 128 B
    static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
    static constexpr uint32_t STAGES = 2;
    static constexpr uint32_t NACC = SX + kSW - 1;         // 7 or 11 shifted accumulators
    static constexpr uint32_t ACC_COLS = NACC * RT;
    static constexpr uint32_t ACC_BUFS = 2 * ACC_COLS <= 512 ? 2 : 1;
    static constexpr uint32_t BUF_STRIDE = 256;            // TMEM column offset of accumulator set 1
    static constexpr uint32_t EPI_BATCH = NACC <= 7 ? 2 : 1;   // 8-row chunks per tcgen05.ld wait (registers)
    static constexpr uint32_t TMEM_COLS = 512;
    // as TcCfg::SPLIT: one set (S_x = 8: 11 x 32 = 352 columns) at alternating bases 0 / B1 (not
    // for S_x = 4, RT = 64: 7 x 64 = 448 columns overlap in 384, the first part would be 6 of 7)
#ifdef NIMBUS_NO_SPLIT
    static constexpr bool SPLIT = false;
#else
    static constexpr bool SPLIT = ACC_BUFS == 1 && ACC_COLS < TMEM_COLS && SX == 8;
#endif
    static constexpr uint32_t B1 = TMEM_COLS - ACC_COLS;
    static constexpr uint32_t LO_A = B1 / RT;                              // base 0: acc_LO_A.. overlap
    static constexpr uint32_t HI_B = (ACC_COLS - B1 + RT - 1) / RT;        // base B1: acc_0..HI_B-1 overlap
    static constexpr uint32_t EPI_WARPS = 8;
    static constexpr uint32_t THREADS = 128 + 32 * EPI_WARPS;
    static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 256;
    static_assert(ACC_COLS <= TMEM_COLS && (ACC_BUFS == 1 || ACC_COLS <= BUF_STRIDE), "TMEM");
    static_assert(RT % 16 == 0 && (RT / 2) % 8 == 0, "epilogue halves of whole 8-row chunks");
    static_assert(SMEM <= 232448, "shared memory");
};

template <int SX, int RT>
__global__ void __launch_bounds__(TCfgT<SX, RT>::THREADS, 1)
k_cop_tc_t(Rns R, const uint8_t* __restrict__ Xt, const uint8_t* __restrict__ Et, uint32_t k, uint32_t RTt,
           uint32_t CT, uint32_t KB, uint32_t ncol, uint32_t* __restrict__ C) {
    using Cfg = TCfgT<SX, RT>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;        // [ACC_BUFS]
    uint64_t* tempty = tfull + 2;                 // [ACC_BUFS]; SPLIT: [0] = a tile's first-part release
    uint64_t* trel = tempty + 2;                  // SPLIT: full release of a tile, by tile parity
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(trel + 2);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nunits = RTt * CT;
    if (threadIdx.x == 0) TRACE(0);
    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < Cfg::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (uint32_t b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1); mbar_init(&tempty[b], Cfg::EPI_WARPS); mbar_init(&trel[b], Cfg::EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) TRACE(1);
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer
            const uint64_t pol_x = policy_evict_last();
            const uint64_t pol_e = policy_evict_last();   // an E tile is reused by every row tile (L2)
            uint32_t it = 0;
            bool waited = false;
            for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x) {
                const uint32_t rt = u % RTt, ct = u / RTt;
                for (uint32_t kb = 0; kb < KB; kb++, it++) {
                    const uint32_t s = it % Cfg::STAGES, ph = (it / Cfg::STAGES) & 1;
                    if (it >= Cfg::STAGES) mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* sa = smem + s * Cfg::STAGE;
                    mbar_arrive_expect_tx(&full[s], Cfg::STAGE);
                    bulk_g2s(sa, Et + ((size_t)ct * KB + kb) * Cfg::A_BYTES, Cfg::A_BYTES, &full[s], pol_e);
                    if (!waited) { pdl_wait(); waited = true; TRACE(2); }
                    bulk_g2s(sa + Cfg::A_BYTES, Xt + ((size_t)rt * KB + kb) * Cfg::B_BYTES, Cfg::B_BYTES, &full[s],
                             pol_x);
                }
            }
        }
    } else if (warp == 1) {
        {   // the whole warp, converged: one elected lane issues (warp-uniform operands)
            // ---------------- MMA issuer
            constexpr uint32_t idesc_full = idesc_i8(Cfg::BM, Cfg::SX * Cfg::RT);         // N = 256
            constexpr uint32_t idesc_lo = idesc_i8(Cfg::BM, (Cfg::SX - 1) * Cfg::RT);     // N = 192
            constexpr uint32_t idesc_one = idesc_i8(Cfg::BM, Cfg::RT);                    // N = 64
            uint32_t it = 0, ti = 0;
            for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ti++) {
                const uint32_t buf = Cfg::ACC_BUFS == 2 ? (ti & 1) : 0;
                const uint32_t use = Cfg::ACC_BUFS == 2 ? (ti >> 1) : ti;
                uint32_t dacc;
                if constexpr (Cfg::SPLIT) {
                    if (ti >= 1) mbar_wait(&tempty[0], (ti - 1) & 1);            // previous tile's overlap drained
                    if (ti >= 2) mbar_wait(&trel[ti & 1], ((ti - 2) >> 1) & 1);  // same-base tile fully drained
                    dacc = tmem + (ti & 1) * Cfg::B1;
                } else {
                    if (use >= 1) mbar_wait(&tempty[buf], (use - 1) & 1);
                    dacc = tmem + buf * Cfg::BUF_STRIDE;
                }
                TRACE(4 + 4 * ti);
                tc_fence_after();
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
                        for (uint32_t j = 0; j < kSW; j++) {
                            const uint64_t ad = sdesc_kmajor_sw128(a0 + j * Cfg::BM * Cfg::BK + kk * 32);
                            if ((kb | kk) != 0 || j == 0) {
                                mma_i8_ss_w(dacc + j * Cfg::RT, ad, bd, idesc_full, (kb | kk) != 0);
                            } else {
                                // first k-step, j >= 1: acc_j..acc_{j+SX-2} exist, acc_{j+SX-1} is new
                                mma_i8_ss_w(dacc + j * Cfg::RT, ad, bd, idesc_lo, 1u);
                                const uint64_t bd3 = sdesc_kmajor_sw128(b0 + (Cfg::SX - 1) * Cfg::RT * Cfg::BK + kk * 32);
                                mma_i8_ss_w(dacc + (j + Cfg::SX - 1) * Cfg::RT, ad, bd3, idesc_one, 0u);
                            }
                        }
                    }
                    mma_commit_w(&empty[s]);
                }
                mma_commit_w(&tfull[buf]);
                TRACE(5 + 4 * ti);
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: lane = coefficient column, 8 rows per tcgen05.ld
        const uint32_t ew = warp - 4;
        const uint32_t sub = ew & 3, half = ew >> 2;
        constexpr uint32_t HR = Cfg::RT / 2, CH = HR / 8, B = Cfg::EPI_BATCH;   // rows per half, chunks
        uint32_t ti = 0;
        for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ti++) {
            const uint32_t rt = u % RTt, ct = u / RTt;
            const uint32_t buf = Cfg::ACC_BUFS == 2 ? (ti & 1) : 0;
            const uint32_t use = Cfg::ACC_BUFS == 2 ? (ti >> 1) : ti;
            mbar_wait(&tfull[buf], use & 1);
            if (ew == 0 && lane == 0) TRACE(6 + 4 * ti);
            tc_fence_after();
            const uint32_t col = ct * Cfg::BM + sub * 32 + lane;
            const uint32_t limb = (col / R.N) % R.L;
            const uint32_t p = R.p[limb], c32 = R.c32[limb];
            if constexpr (Cfg::SPLIT) {
                const uint32_t tb = tmem + ((sub * 32) << 16) + (ti & 1) * Cfg::B1 + half * HR;
                const uint32_t row0 = rt * Cfg::RT + half * HR;
                if ((ti & 1) == 0)
                    epilogue_t_split<Cfg::NACC, Cfg::RT, CH, Cfg::LO_A, Cfg::NACC>(R, tb, row0, col, limb, k, ncol, C,
                                                                                &tempty[0], &trel[0]);
                else
                    epilogue_t_split<Cfg::NACC, Cfg::RT, CH, 0, Cfg::HI_B>(R, tb, row0, col, limb, k, ncol, C,
                                                                        &tempty[0], &trel[1]);
                if (ew == 0 && lane == 0) TRACE(7 + 4 * ti);
                continue;
            }
            const uint32_t tbase = tmem + ((sub * 32) << 16) + buf * Cfg::BUF_STRIDE + half * HR;
#pragma unroll 1
            for (uint32_t c0 = 0; c0 < CH; c0 += B) {
                uint32_t v[B][Cfg::NACC][8];
#pragma unroll
                for (uint32_t b = 0; b < B; b++)
#pragma unroll
                    for (uint32_t s = 0; s < Cfg::NACC; s++) tmem_ld8(tbase + s * Cfg::RT + (c0 + b) * 8, v[b][s]);
                tmem_ld_wait();
                if (c0 + B >= CH) acc_release(&tempty[buf]);      // last chunk in registers
#pragma unroll
                for (uint32_t b = 0; b < B; b++) {
#pragma unroll
                    for (uint32_t q = 0; q < 8; q++) {
                        const uint32_t row = rt * Cfg::RT + half * HR + (c0 + b) * 8 + q;
                        // s < 4 exact (< 2^55), s >= 4 as acc_s (2^(8s) mod p): the sum stays < 2^64
                        uint64_t x = mad_wide(v[b][1][q], 1u << 8, v[b][0][q]);
                        x = mad_wide(v[b][2][q], 1u << 16, x);
                        x = mad_wide(v[b][3][q], 1u << 24, x);
#pragma unroll
                        for (uint32_t s = 4; s < Cfg::NACC; s++) x = mad_wide(v[b][s][q], R.pow8[limb][s], x);
                        if (row < k && col < ncol) C[(size_t)row * ncol + col] = reduce64_pm(x, p, c32);
                    }
                }
            }
            if (ew == 0 && lane == 0) TRACE(7 + 4 * ti);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TRACE(3);
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, Cfg::TMEM_COLS);
    }
}

// ------------------------------------------------------------------ launchers
template <int SX, int CL, int BN>
static cudaError_t launch_sx(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k, uint32_t* d_C,
                             cudaStream_t st) {
    using Cfg = TcCfg<SX, BN>;
    {
        cudaError_t e = ensure_smem(c, k_cop_tc<SX, CL, BN>, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    const uint32_t CT = col_tiles(c, BN), Mt = (k + kBM - 1) / kBM;
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
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cop_tc<SX, CL, BN>, c->rns, d_Xt, (const uint8_t*)w->d_Et, k, Mt,
                                       CT, w->KB, ncol, d_C);
    c->launches++;
    snprintf(c->last_contraction, sizeof(c->last_contraction), "k_cop_tc<%d, %d, %d>", SX, CL, BN);
    return e;
}

static cudaError_t launch_res(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k, uint32_t* d_C,
                              cudaStream_t st) {
    if (c->res_ring == 2) {
        cudaError_t e = ensure_smem(c, k_cop_tc_res2, ResCfg2::SMEM);
        if (e != cudaSuccess) return e;
        const uint32_t ncol = 2 * c->rns.L * c->rns.N;
        const uint32_t CT = col_tiles(c, kBNR);
        const uint32_t grid = CT < (uint32_t)c->num_sms ? CT : (uint32_t)c->num_sms;
        e = launch_pdl(k_cop_tc_res2, dim3(grid), dim3(ResCfg2::THREADS), ResCfg2::SMEM, st, c->rns, d_Xt,
                       (const uint8_t*)w->d_Et, k, CT, w->KB, ncol, d_C);
        c->launches++;
        snprintf(c->last_contraction, sizeof(c->last_contraction), "k_cop_tc_res2");
        return e;
    }
    ResJobs J;
    J.nj = 1;
    J.Et[0] = w->d_Et;
    J.C[0] = d_C;
    return launch_res_jobs(c, J, w->KB, d_Xt, k, st);
}

// The one-shot hint of nimbus_cop_prefetch_next as the kernel's ResPf: where the next resident-X
// contraction's CTAs start (the same k assumed; a wrong guess only prefetches tiles that come later).
static ResPf take_prefetch_hint(nimbus_ctx* c, uint32_t k) {
    ResPf pf;
    {   // measurement switch: own tiles [from, from + self) prefetched before the PDL wait
        const char* es = getenv("NIMBUS_PF_SELF");
        const char* ef = getenv("NIMBUS_PF_FROM");
        pf.self = es ? (uint32_t)atoi(es) : 0u;
        pf.from = ef ? (uint32_t)atoi(ef) : 2u;
        const char* ep = getenv("NIMBUS_PF_POL");     // L2 policy of the next-launch prefetch: 0 none, 1 evict_last, 2 evict_normal
        pf.pol = ep ? (uint32_t)atoi(ep) : 0u;
    }
    const nimbus_encw* w = c->pf_next;
    c->pf_next = nullptr;
    if (!w || !w->d_Et || !resident_ok(c, w, k)) return pf;
    const uint32_t CT = col_tiles(c, kBNR);
    pf.base = (const uint8_t*)w->d_Et;
    pf.tile_bytes = w->KB * ResCfg::B_BYTES;
    pf.ntiles = CT;
    pf.NT = c->rns.N / kBNR;
    pf.fuse = fused_r1_ok(c, w, k) ? 1u : 0u;
    const uint32_t units = pf.fuse ? CT / 2 : CT;
    pf.grid = units < (uint32_t)c->num_sms ? units : (uint32_t)c->num_sms;
    const char* env = getenv("NIMBUS_PF_TILES");      // tiles per CTA to prefetch (measurement switch)
    pf.count = env ? (uint32_t)atoi(env) : 2u;      // measured: C3 17.4 -> 17.2 (1) / 16.7 (2, 3) us, C2 20.1 -> 19.6 / 19.3 / 20.6
    return pf;
}

// the resident-X contraction over up to 4 matmuls sharing X (same m, ell <= 16, k <= 128)
cudaError_t launch_res_jobs(nimbus_ctx* c, const ResJobs& J, uint32_t KB, const uint8_t* d_Xt, uint32_t k,
                            cudaStream_t st) {
    cudaError_t e = ensure_smem(c, k_cop_tc_res<false>, ResCfg::SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    const uint32_t CT = col_tiles(c, kBNR), tiles = CT * J.nj;
    const uint32_t grid = tiles < (uint32_t)c->num_sms ? tiles : (uint32_t)c->num_sms;
    e = launch_pdl(k_cop_tc_res<false>, dim3(grid), dim3(ResCfg::THREADS), ResCfg::SMEM, st, c->rns, d_Xt, J, k, CT, KB,
                   ncol, FuseOut{}, take_prefetch_hint(c, k));
    c->launches++;
    snprintf(c->last_contraction, sizeof(c->last_contraction), "k_cop_tc_res<0>");
    return e;
}

bool resident_ok(const nimbus_ctx* c, const nimbus_encw* w, uint32_t k) {
    return w->bn == kBNR && sx_of(c->rns.ell) == 2 && k <= kBM && w->KB <= kResMaxKB;
}

bool fused_r1_ok(const nimbus_ctx* c, const nimbus_encw* w, uint32_t k) {
    return c->fuse_r1 && c->res_ring == 1 && resident_ok(c, w, k) && c->rns.L == 2 && c->rns.L_out == 1 &&
           2 * w->n > c->rns.N && c->rns.N % (2 * kBNR) == 0;
}

cudaError_t launch_cop_fused_r1(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k, uint64_t seed,
                                uint32_t* d_cts, uint32_t* d_R, cudaStream_t st) {
    if (!fused_r1_ok(c, w, k)) return cudaErrorInvalidValue;
    cudaError_t e = ensure_smem(c, k_cop_tc_res<true>, ResCfg::SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    const uint32_t CT = col_tiles(c, kBNR), P = CT / 2;       // (component, J-tile) pairs
    const uint32_t grid = P < (uint32_t)c->num_sms ? P : (uint32_t)c->num_sms;
    const FuseOut fo{d_cts, d_R, prg_key(seed, 6), w->n};
    ResJobs J;
    J.nj = 1;
    J.Et[0] = w->d_Et;
    e = launch_pdl(k_cop_tc_res<true>, dim3(grid), dim3(ResCfg::THREADS), ResCfg::SMEM, st, c->rns, d_Xt, J, k, CT,
                   w->KB, ncol, fo, take_prefetch_hint(c, k));
    c->launches++;
    {   // writes the ciphertexts and R, and triggers its dependents early
        const void* op[2] = {d_cts, d_R};
        const size_t ob[2] = {(size_t)k * 2 * c->rns.N * 4, (size_t)k * w->n * 4};
        pdl_outputs_set(st, op, ob, 2);
    }
    snprintf(c->last_contraction, sizeof(c->last_contraction), "k_cop_tc_res<1>");
    return e;
}

template <int SX, int RT>
static cudaError_t launch_t(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k, uint32_t* d_C,
                            cudaStream_t st) {
    using Cfg = TCfgT<SX, RT>;
    {
        cudaError_t e = ensure_smem(c, k_cop_tc_t<SX, RT>, Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    const uint32_t CT = col_tiles(c, kBNW), RTt = (k + Cfg::RT - 1) / Cfg::RT;
    const uint32_t nunits = CT * RTt;
    const uint32_t grid = nunits < (uint32_t)c->num_sms ? nunits : (uint32_t)c->num_sms;
    cudaError_t e = launch_pdl(k_cop_tc_t<SX, RT>, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM, st, c->rns, d_Xt,
                               (const uint8_t*)w->d_Et, k, RTt, CT, w->KB, ncol, d_C);
    c->launches++;
    snprintf(c->last_contraction, sizeof(c->last_contraction), "k_cop_tc_t<%d, %d>", SX, RT);
    return e;
}

template <int SX, int BN>
static cudaError_t launch_cl(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k, uint32_t* d_C,
                             cudaStream_t st) {
    return c->cluster == 2 ? launch_sx<SX, 2, BN>(c, w, d_Xt, k, d_C, st) : launch_sx<SX, 1, BN>(c, w, d_Xt, k, d_C, st);
}

// X rows per tile of the transposed kernel (the slice layout follows it): 32 at S_x = 8;
// at S_x = 4, 64 (one accumulator set, N = 256) unless NIMBUS_T_RT=32 (two sets, the
// epilogue overlapped: C5 115.5 vs 108.3 ms -- the extra fill per MAC costs more)
uint32_t transposed_rows(const nimbus_ctx* c) {
    if (sx_of(c->rns.ell) == 8) return 32;
    if (sx_of(c->rns.ell) == 2) return 64;       // 5 accumulators x 64 rows, N = 128
    const char* env = getenv("NIMBUS_T_RT");     // read per call: the slice and the kernel agree
    return env && atoi(env) == 32 ? 32 : 64;
}

cudaError_t launch_cop_tcgen05(nimbus_ctx* c, const nimbus_encw* w, const uint8_t* d_Xt, uint32_t k,
                               uint32_t* d_C, cudaStream_t st) {
    const uint32_t SX = sx_of(c->rns.ell);
    if (!(w->bn == kBNR && resident_ok(c, w, k) && c->res_ring != 2))
        c->pf_next = nullptr;                     // a prefetch hint is for the next launch only
    if (w->bn == kBNW) {
        if (SX == 4) return transposed_rows(c) == 32 ? launch_t<4, 32>(c, w, d_Xt, k, d_C, st)
                                                     : launch_t<4, 64>(c, w, d_Xt, k, d_C, st);
        if (SX == 8) return launch_t<8, 32>(c, w, d_Xt, k, d_C, st);
        if (SX == 2) return launch_t<2, 64>(c, w, d_Xt, k, d_C, st);
        return cudaErrorInvalidValue;
    }
    if (SX == 8) return cudaErrorInvalidValue;    // 8 slices only in the transposed orientation
    if (w->bn == kBNR) {
        if (resident_ok(c, w, k)) return launch_res(c, w, d_Xt, k, d_C, st);
        switch (SX) {
            case 1: return launch_cl<1, kBNR>(c, w, d_Xt, k, d_C, st);
            case 2: return launch_cl<2, kBNR>(c, w, d_Xt, k, d_C, st);
            default: return launch_cl<4, kBNR>(c, w, d_Xt, k, d_C, st);
        }
    }
    switch (SX) {
        case 1: return launch_cl<1, kBNT>(c, w, d_Xt, k, d_C, st);
        case 2: return launch_cl<2, kBNT>(c, w, d_Xt, k, d_C, st);
        default: return launch_cl<4, kBNT>(c, w, d_Xt, k, d_C, st);
    }
}

}  // namespace nimbus
