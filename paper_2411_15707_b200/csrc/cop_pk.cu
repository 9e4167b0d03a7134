// cop_pk.cu -- K5 + K7 fused: the COP contraction computed directly in the PACKED
// output layout, with the mod-switch and the mask in its epilogue (ell in (16, 32],
// n a multiple of 128, Enc(W) in the 128-column "transposed" layout).
//
// RShift packing (stride n: PAPER.md:243) is linear in the rows:
//     c~[theta] = sum_{r<R} X^{r n} c[theta R + r]
//               = sum_{r<R} sum_beta x[theta R + r, beta] X^{r n} Enc(W_beta)
// so, per (component, limb) and output coefficient J,
//     c~[theta][J] = sum_{r<R} sgn(r, J) sum_beta x[theta R + r, beta] E[beta][(J - r n) mod N]
// with sgn = -1 exactly when J < r n (the negacyclic wrap, X^N = -1).  That is a GEMM
// with K = (r, beta) (R m terms) and M = the packed ciphertexts theta -- the same MACs
// as the row-wise contraction (k m 2 L N), but the unpacked C (k x 2LN, 403 MB per C5
// matmul) is never written and no pack kernel reads it back.
//
// When n % 128 == 0 every shift r n is a whole number of 128-coefficient tiles, so the
// operand of term r for output tile T is simply Enc(W) tile (T - r n / 128) mod (N/128),
// and the sign is constant over the tile (wrapped iff 128 T < r n).  The sign cannot be
// applied inside an unsigned int8 MMA; instead a wrapped term multiplies the bitwise
// complement ~x = (2^(8 S_x) - 1) - x, and the epilogue subtracts the precomputed
//     corr[J] = (2^(8 S_x) - 1) * sum_{r: J < r n} ColSum[(J - r n) mod N]   (mod p),
// ColSum[col] = sum_beta E[beta][col]: sum_beta ~x E = (2^(8S_x)-1) ColSum - sum_beta x E.
// Rows theta R + r >= k_q ("pad with zeros") are x = 0, i.e. ~x = all ones
// in the complemented copy, so corr is the same for every theta.
//
// Exactness: 8-bit slices as in cop_tc.cu (acc_s = sum_{i+j=s} x_i e_j in int32 TMEM);
// the K loop runs in chunks of at most 64 k-blocks (8192 terms: acc_s < 4 * 8192 * 255^2
// < 2^31, and the recombination sum_s acc_s (2^(8s) mod p) < 2^63), each chunk drained
// by the epilogue into a running residue mod p.
//
// Work unit = (matmul, limb pass, component, theta tile of RT packed ciphertexts,
// 128-coefficient J tile).  The limb passes of a matmul run in the order L-1 .. L_out
// (the limbs ModDown drops) then 0 .. L_out-1, so that the Enc(W) blocks in use at any
// time belong to one (component, limb) slab (25 MB at m = 768, 100 MB at m = 3072) and
// stay in L2 while the R shifted output tiles and the theta tiles that read each block
// come by.  A dropped-limb pass leaves its centred residues rho in an L2-resident
// scratch and raises a per-tile flag; the output passes wait for the flag and apply
// ModDown (c_i <- (c_i - [c_l]) p_l^-1) and the mask
// b -= Emb_{q'}(r) (§8(c) #13) in the epilogue, which writes the compact
// output ciphertexts and R.  Units are handed out in order by an atomic counter (the
// CTAs in flight always work on neighbouring units); one persistent launch serves a
// whole job list (the 72 matmuls of the C5 pass), so there is one tail per pass.
#include <memory>
#include <vector>
#include <cstdio>
#include <cstring>
#include "internal.h"
#include "slice_dev.cuh"

namespace nimbus {

constexpr uint32_t kPkMaxJobs = 128;
constexpr uint32_t kPkMaxChunkKB = 64;     // k-blocks (x 128 terms) per accumulator drain at S_x <= 4
constexpr uint32_t kPkQ = 4;               // unit-id queue depth (producer -> MMA issuer, epilogue)

struct PkJob {
    const uint8_t* Et;        // Enc(W) tiles [ct][kb][4 planes][128][128 B]
    const uint8_t* Xp;        // packed X slices [(r, cmp)][theta tile][kb][S_x][RT][128 B]
    const uint32_t* corr;     // [comp][limb][N]
    uint32_t* cts;            // [theta_global][comp][L_out][N]
    uint32_t* Rout;           // [alpha_global][n], or null
    const uint32_t* X;        // slice kernel input [k][m]
    int32_t* rho;             // [drop][theta tile row][comp][N]: centred residues of the dropped limbs
    uint32_t* flags;          // [drop][comp][theta tile][J tile]: rho written
    uint64_t key;             // prg_key(mask_seed, 6)
    uint32_t m, KB, Rr, n, kq, nct, ntheta, TT, CKB, NCH, nflags;
    uint32_t ws, wc;          // unit order: shift in tiles (n / 128 mod NT) and its cycle length; wc = 0: T fastest
    uint32_t unit_end;        // contraction: prefix end of this job's units
    uint32_t blk_end;         // slice kernel: prefix end of this job's blocks
};
struct PkParams {
    uint32_t njobs;
    uint32_t* ctr;            // unit dispatch counter (zeroed by the slice kernel)
    uint32_t epol;            // L2 policy of the Enc(W) copies: 0 evict_last, 1 evict_normal, 2 evict_first
#ifdef NIMBUS_PK_DIAG
    uint32_t diag;            // diagnostic build only (wrong results): 1 every X copy reads the job's first block,
                              // 2 every Enc(W) copy the slab's first tile -- what each stream costs in DRAM bytes
#endif
    PkJob job[kPkMaxJobs];
};

#ifdef NIMBUS_TRACE
// Debug-only cycle accounting per CTA (tools/pk_stats.py): [0] MMA warp waiting for drained
// accumulators, [1] waiting for X, [2] waiting for Enc(W), [3] MMA warp total, [4] epilogue in
// drains, [5] epilogue in finalize, [6] epilogue waiting for accumulators, [7] units,
// [8] epilogue waiting for flags/rho prefetch, [9] producer waiting for free slots.
__device__ unsigned long long* g_pk_stats = nullptr;
extern "C" int nimbus_pk_stats_set(void* p) { return (int)cudaMemcpyToSymbol(g_pk_stats, &p, sizeof(p)); }
#define PKS_T0(v) const long long v = clock64()
#define PKS_ADD(i, t0) do { pks[i] += (unsigned long long)(clock64() - (t0)); } while (0)
#define PKS_INC(i) do { pks[i] += 1ull; } while (0)
#define PKS_DECL unsigned long long pks[16] = {0}
#define PKS_FLUSH do { if (g_pk_stats && lane == 0) for (int i_ = 0; i_ < 16; i_++) if (pks[i_]) \
        atomicAdd(&g_pk_stats[blockIdx.x * 16 + i_], pks[i_]); } while (0)
#else
#define PKS_DECL do { } while (0)
#define PKS_FLUSH do { } while (0)
#define PKS_T0(v) do { } while (0)
#define PKS_ADD(i, t0) do { } while (0)
#define PKS_INC(i) do { } while (0)
#endif

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                    "r"(v[7]) : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                 :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]) : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }   // the 8 epilogue warps
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// Shared memory: two rings with their own barriers, so a freed slot is refilled after a
// quarter (E) / one (X) k-step of MMAs instead of a whole one: an Enc(W) ring of ESLOTS
// slots holding ONE byte plane (128 columns x 128 B = 16 KB) each, and an X ring of XSLOTS
// slots holding the S_x slices of one (term r, k-block).  A 2-slot ring of whole
// (E + X) k-steps left the MMA issuer waiting for data ~25% of the time (L2 latency).
//
// P2 (CTA pairs, tcgen05 cta_group::2): the pair's MMA is M = 256 -- two neighbouring J tiles, CTA
// r holding the Enc(W) plane of tile 2P + r -- over ONE theta tile whose X block is split by rows
// (the MMA's N): CTA r holds slices [r S_x/2, (r+1) S_x/2).  Each SM then reads its A half and its
// B half per MMA instead of a whole B, and fills half the X: the single-CTA / multicast form reads
// A 4 KB + B 6.5 KB per 104-cycle MMA and fills 54 B/cycle more, above the 128 B/cycle of shared
// memory (smem-bound at ~0.82 of the tensor rate); the pair form needs ~110 B/cycle.
template <int SX, int RT, bool P2 = false>
struct PkCfg {
    static constexpr uint32_t BM = kBNW, BK = kBK;
    static constexpr uint32_t A_BYTES = kSW * BM * BK;     // 64 KB: 4 planes x 128 columns x 128 B
    static constexpr uint32_t P_BYTES = BM * BK;           // one plane: 16 KB
    static constexpr uint32_t B_BYTES = SX * RT * BK;      // S_x slices x RT rows x 128 B
    static constexpr uint32_t XB = P2 ? B_BYTES / 2 : B_BYTES;   // this CTA's part of an X block
    // S_x = 2 (ell <= 16) issues half the MMA work per Enc(W) plane, so its planes are consumed twice
    // as fast, and P2 halves the X slots: two more Enc(W) slots in flight
    static constexpr uint32_t ESLOTS = (SX == 2 || P2) ? 10 : 8, XSLOTS = 3;
    static constexpr uint32_t OFF_X = ESLOTS * P_BYTES;
    static constexpr uint32_t RING = OFF_X + XSLOTS * XB;
    static constexpr uint32_t NACC = SX + kSW - 1;
    static constexpr uint32_t ZCOL = 480;                  // TMEM columns [480, 488): a zero A operand
    static constexpr uint32_t NCHK = (RT + 7) / 8;         // 8-row chunks of an accumulator (the last may hold 4)
    static constexpr uint32_t TAIL = RT - 8 * (NCHK - 1);  // rows of the last chunk: 8, or 4 (RT = 52)
    static constexpr uint32_t CPT0 = (NCHK + 1) / 2;       // chunks of the first epilogue half
    static constexpr uint32_t EPI_WARPS = 8;
    static constexpr uint32_t THREADS = 128 + 32 * EPI_WARPS;
    static constexpr size_t SMEM = (size_t)RING + 1024 + 512;     // alignment slack + barriers, queue
    static_assert(RT % 4 == 0 && (TAIL == 8 || TAIL == 4), "8-row chunks, a 4-row tail at most");
    static_assert((SX * RT) % 16 == 0 && SX * RT <= 256, "MMA N");
    static_assert(NACC * RT <= ZCOL, "TMEM: accumulators below the zero operand");
    static_assert(SX == 2 || SX == 4, "packed contraction: 2 or 4 X slices");
    static_assert(XB % 1024 == 0, "swizzle atoms");
    // cta_group::2 kind::i8 takes N in steps of 16 (N = 208, RT = 52, checked bit-exact on B200)
    static_assert(!P2 || (SX * RT) % 16 == 0, "cta_group::2 kind::i8: N a multiple of 16");
    static_assert(SMEM <= 232448, "shared memory");
};

// cluster-unit u -> (job, limb pass, component, group of CL theta tiles, J tile); T fastest so
// that the clusters in flight read neighbouring Enc(W) tiles of one (component, limb) slab.
// The CL CTAs of a cluster take theta tiles g CL + rank of the same (job, pass, comp, T): they
// consume the same Enc(W) planes in lockstep, each plane fetched once and multicast to all.
struct PkUnit {
    uint32_t j, pass, comp, tt, T;
};
// j: the caller's job cursor -- a CTA receives its units in increasing order, so the job search
// resumes where the previous unit's ended (a scan from job 0 per unit cost ~8% of the pass)
// P2: the pair takes J tiles 2 Tp + rank of one theta tile instead.
__device__ __forceinline__ PkUnit pk_decode(const PkParams& P, uint32_t u, uint32_t NT, uint32_t CL, uint32_t rank,
                                            uint32_t& j, bool p2 = false) {
    PkUnit x;
    while (u >= P.job[j].unit_end) j++;
    uint32_t v = u - (j ? P.job[j - 1].unit_end : 0u);
    x.j = j;
    if (p2) {
        const uint32_t NTp = NT >> 1;
        x.T = (v % NTp) * 2 + rank; v /= NTp;
        x.tt = v % P.job[j].TT; v /= P.job[j].TT;
        x.comp = v & 1;
        x.pass = v >> 1;
        return x;
    }
    const uint32_t G = (P.job[j].TT + CL - 1) / CL;
    if (const uint32_t wc = P.job[j].wc) {
        // theta groups fastest, then the J tiles in shift order: position i of the walk is tile
        // (i mod wc) ws + i / wc, so a unit's R shifted Enc(W) tiles (T - r ws) are the R walk positions
        // before its own and the units in flight read a window of the slab instead of all of it
        x.tt = (v % G) * CL + rank; v /= G;
        const uint32_t i = v % NT; v /= NT;
        x.T = ((i % wc) * P.job[j].ws + i / wc) % NT;
        x.comp = v & 1;
        x.pass = v >> 1;
        return x;
    }
    x.T = v % NT; v /= NT;
    x.tt = (v % G) * CL + rank; v /= G;
    x.comp = v & 1;
    x.pass = v >> 1;
    return x;
}
// limb of pass `pass`: dropped limbs L-1 .. L_out first, then 0 .. L_out-1
__device__ __forceinline__ uint32_t pk_limb(const Rns& R, uint32_t pass) {
    const uint32_t nd = R.L - R.L_out;
    return pass < nd ? R.L - 1 - pass : pass - nd;
}

// mbarrier wait with cluster-scope acquire (the phase may be completed by the peer CTA)
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONEC_%=;\n\t"
        "bra WAITC_%=;\n\t"
        "DONEC_%=:\n\t}"
        :: "r"(smem_u32(bar)), "r"(parity), "r"(0x989680) : "memory");
}
__device__ __forceinline__ uint32_t mapa_cl(uint32_t saddr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(cta));
    return r;
}
// arrive on the mbarrier at the same offset in CTA `cta` of the cluster (release, cluster scope)
__device__ __forceinline__ void mbar_arrive_cl(uint64_t* bar, uint32_t cta) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(mapa_cl(smem_u32(bar), cta))
                 : "memory");
}
// the same without release semantics: the P2 relay publishes no writes of its own (the bulk copies it
// reports are complete at its local barrier), and a release per arrive serialises the relay thread
__device__ __forceinline__ void mbar_arrive_cl_relaxed(uint64_t* bar, uint32_t cta) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" :: "r"(mapa_cl(smem_u32(bar), cta))
                 : "memory");
}
__device__ __forceinline__ void st_cl_u32(uint32_t* p, uint32_t cta, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(mapa_cl(smem_u32(p), cta)), "r"(v) : "memory");
}

// ---- tcgen05 with cta_group::2 (P2: every tcgen05 instruction of the kernel uses the pair form)
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(dst_smem)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void mma2_i8_ss_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void mma2_i8_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
        :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// arrive on the mbarrier at this offset in both CTAs of the pair when the pair's MMAs complete
__device__ __forceinline__ void mma2_commit_w(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
        :: "r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}

template <int SX, int RT, int CL, bool P2 = false>
__global__ void __launch_bounds__(PkCfg<SX, RT, P2>::THREADS, 1)
k_cop_pk(const __grid_constant__ Rns R, const __grid_constant__ PkParams P, uint32_t total_units) {
    using Cfg = PkCfg<SX, RT, P2>;
    static_assert(!P2 || CL == 2, "P2: CTA pairs");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* efull = reinterpret_cast<uint64_t*>(smem + Cfg::RING);
    uint64_t* eempty = efull + Cfg::ESLOTS;
    uint64_t* xfull = eempty + Cfg::ESLOTS;
    uint64_t* xempty = xfull + Cfg::XSLOTS;
    uint64_t* tfull = xempty + Cfg::XSLOTS;
    uint64_t* tempty = tfull + 1;
    uint64_t* qfull = tempty + 1;                 // [kPkQ]
    uint64_t* qempty = qfull + kPkQ;              // [kPkQ]
    uint32_t* unit_q = reinterpret_cast<uint32_t*>(qempty + kPkQ);
    uint32_t* tmem_slot = unit_q + kPkQ;

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CL > 1 ? cluster_ctarank() : 0;
    PKS_DECL;
    const uint32_t N = R.N, NT = N / Cfg::BM, L = R.L, ND = R.L - R.L_out;
    constexpr uint32_t MASK = (1u << CL) - 1;
    // P2: the leader's full barriers also wait for the peer's copies (relayed by the peer's warp 1),
    // its tempty for both CTAs' epilogues; the pair's commits arrive on both CTAs' empty barriers
    const uint32_t nfull = P2 && rank == 0 ? 2 : 1;
    if (warp == 0 && lane == 0) {
        for (uint32_t s = 0; s < Cfg::ESLOTS; s++) { mbar_init(&efull[s], nfull); mbar_init(&eempty[s], P2 ? 1 : CL); }
        for (uint32_t s = 0; s < Cfg::XSLOTS; s++) { mbar_init(&xfull[s], nfull); mbar_init(&xempty[s], 1); }
        mbar_init(tfull, 1);
        mbar_init(tempty, Cfg::EPI_WARPS * nfull);
        // unit ids come from the cluster's leader; its queue slot is free once every consumer of
        // every CTA has read it (MMA warp + epilogue warps, and the peers' producers)
        for (uint32_t q = 0; q < kPkQ; q++) {
            mbar_init(&qfull[q], 1);
            mbar_init(&qempty[q], CL * (1 + Cfg::EPI_WARPS) + (CL - 1));
        }
        fence_mbar_init();
    }
    if constexpr (P2) {
        cluster_sync();                                 // both CTAs running before the pair allocation
        if (warp == 2) tmem_alloc2(tmem_slot, 512);
    } else {
        if (warp == 2) tmem_alloc(tmem_slot, 512);
    }
    tc_fence_before();
    if (CL > 1) cluster_sync(); else __syncthreads();   // the peers' barriers exist before any multicast
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_trigger();
    // a consumer takes unit id i: wait, read, release the leader's queue slot
    auto take_unit = [&](uint32_t i, bool arrive_one) -> uint32_t {
        const uint32_t q = i % kPkQ;
        if (CL > 1) mbar_wait_cl(&qfull[q], (i / kPkQ) & 1); else mbar_wait(&qfull[q], (i / kPkQ) & 1);
        const uint32_t u = unit_q[q];
        if (arrive_one) {
            if (CL > 1 && rank != 0) mbar_arrive_cl(&qempty[q], 0); else mbar_arrive(&qempty[q]);
        }
        return u;
    };

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer: per (kb, r) the X slices of this CTA's theta tile and the 4 byte
            // planes of one Enc(W) block (plane jp fetched by CTA jp % CL, multicast to the cluster)
            // an Enc(W) block serves R output tiles x theta tiles: in the walk order (PkJob::wc) within a few
            // k-steps of one another, so it needs no protection and leaves the evict_last lines to X
            const uint64_t pol_e = P.epol == 0 ? policy_evict_last() : P.epol == 1 ? policy_evict_normal() : policy_evict_first();
            const uint64_t pol_x = policy_evict_last();    // X blocks serve every J tile
            pdl_wait();                                    // X slices, counter and flags: the slice kernel's
            uint32_t ie = 0, ix = 0, jcur = 0;
            for (uint32_t i = 0;; i++) {
                uint32_t u;
                if (rank == 0) {
                    // every unit, the first included, comes from the counter: a unit is only ever held by
                    // a running cluster, so a flag wait never depends on one that has not been scheduled
                    u = atomicAdd(P.ctr, 1u);
                    const uint32_t q = i % kPkQ;
                    if (i >= kPkQ) mbar_wait(&qempty[q], ((i / kPkQ) & 1) ^ 1);
                    unit_q[q] = u;
                    for (uint32_t c = 1; c < (uint32_t)CL; c++) st_cl_u32(&unit_q[q], c, u);
                    mbar_arrive(&qfull[q]);
                    for (uint32_t c = 1; c < (uint32_t)CL; c++) mbar_arrive_cl(&qfull[q], c);
                } else {
                    u = take_unit(i, true);
                }
                if (u >= total_units) break;
                const PkUnit U = pk_decode(P, u, NT, CL, rank, jcur, P2);
                const PkJob& J = P.job[U.j];
                const bool ghost = U.tt >= J.TT;                      // a cluster's spare theta tile
                const uint32_t limb = pk_limb(R, U.pass);
                const size_t slab = ((size_t)U.comp * L + limb) * NT;
                const uint32_t shift_t = J.n / Cfg::BM;               // tiles per shift step
                for (uint32_t kb = 0; kb < J.KB; kb++) {
                    for (uint32_t r = 0; r < J.Rr; r++) {
                        const uint32_t sh = r * shift_t;
                        const bool wrap = U.T < sh;
                        const uint32_t srcT = wrap ? U.T + NT - sh : U.T - sh;
                        {   // X slices of (r, kb)
                            const uint32_t s = ix % Cfg::XSLOTS, ph = (ix / Cfg::XSLOTS) & 1;
                            if (ix >= Cfg::XSLOTS) { PKS_T0(t0); mbar_wait(&xempty[s], ph ^ 1); PKS_ADD(10, t0); }
                            ix++;
                            if (ghost) {
                                mbar_arrive(&xfull[s]);
                            } else {
                                // (P2: this CTA's half of the block; the pair's wrap agrees, n / 128 even)
                                mbar_arrive_expect_tx(&xfull[s], Cfg::XB);
                                size_t xo = ((((size_t)(2 * r + (wrap ? 1 : 0)) * J.TT + U.tt) * J.KB + kb) * Cfg::B_BYTES) +
                                            (P2 ? rank * Cfg::XB : 0u);
#ifdef NIMBUS_PK_DIAG
                                if (P.diag == 1) xo = 0;
#endif
                                bulk_g2s(smem + Cfg::OFF_X + s * Cfg::XB, J.Xp + xo, Cfg::XB, &xfull[s], pol_x);
                            }
                        }
                        const uint8_t* eb = J.Et + ((slab + srcT) * J.KB + kb) * Cfg::A_BYTES;
#ifdef NIMBUS_PK_DIAG
                        if (P.diag == 2) eb = J.Et + (slab * J.KB + kb) * Cfg::A_BYTES;
#endif
                        for (uint32_t jp = 0; jp < kSW; jp++, ie++) {   // the 4 byte planes of the Enc(W) block
                            const uint32_t s = ie % Cfg::ESLOTS, ph = (ie / Cfg::ESLOTS) & 1;
                            // the slot is free in every CTA of the cluster (CL commits)
                            if (ie >= Cfg::ESLOTS) {
                                PKS_T0(t0);
                                if (CL > 1) mbar_wait_cl(&eempty[s], ph ^ 1); else mbar_wait(&eempty[s], ph ^ 1);
                                PKS_ADD(9, t0);
                            }
                            mbar_arrive_expect_tx(&efull[s], Cfg::P_BYTES);
                            if (CL == 1 || P2)      // P2: each CTA its own J tile's plane
                                bulk_g2s(smem + s * Cfg::P_BYTES, eb + jp * Cfg::P_BYTES, Cfg::P_BYTES, &efull[s], pol_e);
                            else if (jp % CL == rank)
                                bulk_g2s_mc(smem + s * Cfg::P_BYTES, eb + jp * Cfg::P_BYTES, Cfg::P_BYTES, &efull[s],
                                            MASK, pol_e);
                        }
                    }
                }
            }
        }
    } else if (warp == 1 && P2 && rank != 0) {
        // ---------------- P2 peer: relay.  The pair's MMAs read this CTA's Enc(W) planes and X half,
        // so the leader's full barriers must also see this CTA's copies land: in the producer's order,
        // wait for each local full barrier and arrive on the leader's (release, cluster scope)
        uint32_t ie = 0, ix = 0, jcur = 0;
        for (uint32_t i = 0;; i++) {
            const uint32_t u = take_unit(i, false);
            __syncwarp();
            if (lane == 0) mbar_arrive_cl(&qempty[i % kPkQ], 0);
            if (u >= total_units) break;
            const PkUnit U = pk_decode(P, u, NT, CL, rank, jcur, P2);
            const uint32_t KB = P.job[U.j].KB, Rr = P.job[U.j].Rr;
            if (lane == 0) {
                for (uint32_t kb = 0; kb < KB; kb++) {
                    for (uint32_t r = 0; r < Rr; r++, ix++) {
                        mbar_wait(&xfull[ix % Cfg::XSLOTS], (ix / Cfg::XSLOTS) & 1);
                        mbar_arrive_cl_relaxed(&xfull[ix % Cfg::XSLOTS], 0);
                        for (uint32_t jp = 0; jp < kSW; jp++, ie++) {
                            mbar_wait(&efull[ie % Cfg::ESLOTS], (ie / Cfg::ESLOTS) & 1);
                            mbar_arrive_cl_relaxed(&efull[ie % Cfg::ESLOTS], 0);
                        }
                    }
                }
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (the whole warp, converged; one elected lane issues):
        // D[coefficient][theta] += E_j^T . [x_0 | x_1 | .. ] per plane j.  Descriptors are the slot
        // base descriptors plus (kk * 32 B) >> 4 in the start-address field.  P2: the leader issues
        // the pair's M = 256 MMAs (A: each CTA's plane, B: each CTA's half of the X block, D: each
        // CTA's 128 coefficient lanes x all S_x RT columns -- the same accumulator layout).
        constexpr uint32_t idesc = idesc_i8(P2 ? 2 * Cfg::BM : Cfg::BM, SX * RT);
        const uint64_t e_desc0 = sdesc_kmajor_sw128(smem_u32(smem));
        const uint64_t x_desc0 = sdesc_kmajor_sw128(smem_u32(smem + Cfg::OFF_X));
        constexpr uint64_t EP = Cfg::P_BYTES >> 4, XP = Cfg::XB >> 4;
        uint32_t ie = 0, ix = 0, gc = 0, jcur = 0;
        PKS_T0(t_mma0);
        for (uint32_t i = 0;; i++) {
            const uint32_t u = take_unit(i, false);
            __syncwarp();
            if (lane == 0) {
                if (CL > 1 && rank != 0) mbar_arrive_cl(&qempty[i % kPkQ], 0); else mbar_arrive(&qempty[i % kPkQ]);
            }
            if (u >= total_units) { PKS_ADD(3, t_mma0); break; }
            PKS_INC(7);
            const PkUnit U = pk_decode(P, u, NT, CL, rank, jcur, P2);
            const uint32_t KB = P.job[U.j].KB, Rr = P.job[U.j].Rr, CKB = P.job[U.j].CKB, NCH = P.job[U.j].NCH;
            const bool ghost = U.tt >= P.job[U.j].TT;
            for (uint32_t c = 0; c < NCH; c++, gc++) {
                {   // accumulators drained (and zeroed) -- P2: in both CTAs
                    PKS_T0(t0);
                    if (P2) mbar_wait_cl(tempty, gc & 1); else mbar_wait(tempty, gc & 1);
                    PKS_ADD(0, t0);
                }
                tc_fence_after();
                const uint32_t kb1 = min(KB, (c + 1) * CKB);
                for (uint32_t kb = c * CKB; kb < kb1; kb++) {
                    for (uint32_t r = 0; r < Rr; r++, ix++) {
                        const uint32_t xs = ix % Cfg::XSLOTS;
                        {
                            PKS_T0(t0);
                            if (P2) mbar_wait_cl(&xfull[xs], (ix / Cfg::XSLOTS) & 1);
                            else mbar_wait(&xfull[xs], (ix / Cfg::XSLOTS) & 1);
                            PKS_ADD(1, t0);
                        }
                        const uint64_t bd = x_desc0 + xs * XP;
                        // a chunk starts from zero accumulators without a TMEM clear: 0 . X (A = the zero
                        // operand in TMEM, N = S_x RT columns per MMA) sets acc_S_x..acc_{NACC-1} (S_x = 4: one
                        // MMA at acc_3; S_x = 2: acc_2 and acc_3), plane 0's first MMA (no accumulate) then sets
                        // acc_0..acc_{S_x-1}
                        const bool first = kb == c * CKB && r == 0;
                        if (first && !ghost) {
#pragma unroll
                            for (uint32_t z = SX; z < Cfg::NACC; z += SX) {
                                const uint32_t d = tmem + (z < Cfg::NACC - SX ? z : Cfg::NACC - SX) * RT;
                                if constexpr (P2) mma2_i8_ts_w(d, tmem + Cfg::ZCOL, bd, idesc, 0u);
                                else mma_i8_ts_w(d, tmem + Cfg::ZCOL, bd, idesc, 0u);
                            }
                        }
#pragma unroll
                        for (uint32_t jp = 0; jp < kSW; jp++, ie++) {
                            const uint32_t es = ie % Cfg::ESLOTS;
                            {
                                PKS_T0(t0);
                                if (CL > 1) mbar_wait_cl(&efull[es], (ie / Cfg::ESLOTS) & 1);
                                else mbar_wait(&efull[es], (ie / Cfg::ESLOTS) & 1);
                                PKS_ADD(2, t0);
                            }
                            tc_fence_after();
                            const uint64_t ad = e_desc0 + es * EP;
                            if (!ghost) {
#pragma unroll
                                for (uint32_t kk = 0; kk < Cfg::BK / 32; kk++) {
                                    const uint32_t acc = (first && jp == 0 && kk == 0) ? 0u : 1u;
                                    if constexpr (P2) mma2_i8_ss_w(tmem + jp * RT, ad + 2 * kk, bd + 2 * kk, idesc, acc);
                                    else mma_i8_ss_w(tmem + jp * RT, ad + 2 * kk, bd + 2 * kk, idesc, acc);
                                }
                            }
                            // this plane's slot is free (in every CTA of the cluster) once its MMAs retire
                            if constexpr (P2) mma2_commit_w(&eempty[es]);
                            else if (CL > 1) mma_commit_mc_w(&eempty[es], MASK);
                            else mma_commit_w(&eempty[es]);
                        }
                        if constexpr (P2) mma2_commit_w(&xempty[xs]); else mma_commit_w(&xempty[xs]);
                    }
                }
                if constexpr (P2) mma2_commit_w(tfull); else mma_commit_w(tfull);
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: lane = coefficient column, 8-row chunks of the theta tile
        const uint32_t ew = warp - 4;
        const uint32_t sub = ew & 3, half = ew >> 2;
        constexpr uint32_t CPT = Cfg::CPT0;
        const uint32_t ch0 = half * Cfg::CPT0;
        const uint32_t nch = half ? Cfg::NCHK - Cfg::CPT0 : Cfg::CPT0;     // chunks of this thread
        const uint32_t tl = tmem + ((sub * 32) << 16);
        const uint32_t zero8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        pdl_wait();          // flags / rho / outputs: after the slice kernel (and the stream's earlier work)
        // the zero A operand (8 columns x 128 lanes) the MMA issuer starts every chunk with
        if (half == 0) tmem_st8(tl + Cfg::ZCOL, zero8);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) { if (P2 && rank != 0) mbar_arrive_cl(tempty, 0); else mbar_arrive(tempty); }

        uint32_t acc[CPT][8];        // running residue of the unit's limb (mod p_limb)
        uint32_t gc = 0, jcur = 0;
        for (uint32_t i = 0;; i++) {
            const uint32_t u = take_unit(i, false);
            __syncwarp();
            if (lane == 0) {
                if (CL > 1 && rank != 0) mbar_arrive_cl(&qempty[i % kPkQ], 0); else mbar_arrive(&qempty[i % kPkQ]);
            }
            if (u >= total_units) break;
            const PkUnit U = pk_decode(P, u, NT, CL, rank, jcur, P2);
            const PkJob& J = P.job[U.j];
            const bool ghost = U.tt >= J.TT;
            const uint32_t Jc = U.T * Cfg::BM + sub * 32 + lane;         // output coefficient
            const uint32_t limb = pk_limb(R, U.pass);
            const uint32_t p = R.p[limb], c32 = R.c32[limb];
            // the finalize's operands are fetched before the drains, so their L2 latency hides under
            // the MMAs: the complement correction, and -- for a pass after a dropped limb -- its flag
            // and centred residues
            const uint32_t ndep = (U.pass < ND ? U.pass : ND) * (ghost ? 0 : 1);   // dropped limbs it depends on
            const size_t fl_tile = ((size_t)U.comp * J.TT + U.tt) * NT + U.T;
            const size_t fl_stride = (size_t)2 * J.TT * NT;
            const size_t rho_stride = (size_t)J.TT * RT * 2 * N;
            PKS_T0(t_pre);
            const uint32_t cr = __ldg(J.corr + ((size_t)U.comp * L + limb) * N + Jc);
            int32_t rh0[CPT][8];
            if (ndep) {
                if (ew == 0 && lane == 0) {
                    for (uint32_t d = 0; d < ndep; d++)
                        while (ld_acquire(J.flags + d * fl_stride + fl_tile) == 0) __nanosleep(64);
                }
                epi_bar();
#pragma unroll
                for (uint32_t ci = 0; ci < CPT; ci++)
#pragma unroll
                    for (uint32_t qq = 0; qq < 8; qq++) {
                        const uint32_t row = (ch0 + ci) * 8 + qq;
                        rh0[ci][qq] = 0;
                        // issued here, consumed after the drains (asm volatile: the compiler may not sink the
                        // load to its use, where its L2 latency would stall the finalize)
                        if (ci < nch && row < (uint32_t)RT)
                            asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(rh0[ci][qq])
                                         : "l"(J.rho + ((size_t)(U.tt * RT + row) * 2 + U.comp) * N + Jc));
                    }
            }
            PKS_ADD(8, t_pre);
            for (uint32_t c = 0; c < J.NCH; c++, gc++) {
                { PKS_T0(t0); mbar_wait(tfull, gc & 1); PKS_ADD(6, t0); }
                PKS_T0(t_dr);
                tc_fence_after();
#pragma unroll
                for (uint32_t ci = 0; ci < CPT; ci++) {
                    if (ci >= nch) continue;
                    uint32_t v[Cfg::NACC][8];
                    const uint32_t col = (ch0 + ci) * 8;
                    const bool t4 = Cfg::TAIL == 4 && ch0 + ci == Cfg::NCHK - 1;
                    PKS_T0(t_ld);
                    if (t4) {
#pragma unroll
                        for (uint32_t s2 = 0; s2 < Cfg::NACC; s2++) tmem_ld4(tl + s2 * RT + col, v[s2]);
                    } else {
#pragma unroll
                        for (uint32_t s2 = 0; s2 < Cfg::NACC; s2++) tmem_ld8(tl + s2 * RT + col, v[s2]);
                    }
                    tmem_ld_wait();
                    PKS_ADD(11, t_ld);
#pragma unroll
                    for (uint32_t qq = 0; qq < 8; qq++) {
                        uint64_t x = mad_wide(v[1][qq], 1u << 8, v[0][qq]);
                        x = mad_wide(v[2][qq], 1u << 16, x);
                        x = mad_wide(v[3][qq], 1u << 24, x);
#pragma unroll
                        for (uint32_t s2 = 4; s2 < Cfg::NACC; s2++) x = mad_wide(v[s2][qq], R.pow8[limb][s2], x);
                        const uint32_t red = reduce64_pm(x, p, c32);
                        acc[ci][qq] = c == 0 ? red : addmod(acc[ci][qq], red, p);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {                        // the MMA issuer may start the next chunk
                    if (P2 && rank != 0) mbar_arrive_cl(tempty, 0); else mbar_arrive(tempty);
                }
                PKS_ADD(4, t_dr);
            }
            if (ghost) continue;
            PKS_T0(t_fin);
            // ---- the unit's limb is complete: remove the complement offset, then ModDown / mask / store.
            // Everything per row is incremental (this thread's rows are consecutive packed ciphertexts
            // tg of one column J): the mask PRG counter steps by gamma N.
            const uint32_t tg0 = U.tt * RT + ch0 * 8;
            const bool out_pass = U.pass >= ND, masked = out_pass && U.comp == 0;
            const uint64_t gN = 0x9E3779B97F4A7C15ULL * (uint64_t)N;
            const uint64_t z = J.key + 0x9E3779B97F4A7C15ULL * ((uint64_t)tg0 * N + Jc + 1);
            const uint32_t ri = Jc / J.n, jj = Jc - ri * J.n;             // R column of this J (valid if ri < R)
            const bool r_col = masked && limb == 0 && J.Rout && ri < J.Rr;
            const uint32_t qy = tg0 / J.nct, th = tg0 - qy * J.nct;
            uint32_t* ctsp = J.cts + (((size_t)tg0 * 2 + U.comp) * R.L_out + limb) * N + Jc;
            const size_t cts_row = (size_t)2 * R.L_out * N;
            // chunk loop NOT unrolled (the chunk's residues are selected out of the register arrays):
            // one copy of the row body instead of CPT keeps the kernel's hot code inside the
            // instruction cache (unrolled, ~13% of all warp stalls were instruction fetch).  Within a
            // chunk the 8 rows go stage by stage, each stage branch-free (stores predicated): the unit-
            // uniform decisions sit between stages, so the scheduler interleaves the 8 rows' dependency
            // chains instead of running one row's ~90 dependent instructions at a time
            const uint32_t iv_w = ND ? R.inv_p[L - 1][limb] : 0, iv_sh = ND ? R.inv_p_sh[L - 1][limb] : 0;
#pragma unroll 1
            for (uint32_t ci = 0; ci < nch; ci++) {
                uint32_t v8[8];
                int32_t r8[8];
#pragma unroll
                for (uint32_t qq = 0; qq < 8; qq++) {
                    uint32_t a = acc[0][qq];
                    int32_t r = rh0[0][qq];
#pragma unroll
                    for (uint32_t k = 1; k < CPT; k++) {
                        a = ci == k ? acc[k][qq] : a;
                        r = ci == k ? rh0[k][qq] : r;
                    }
                    v8[qq] = submod(a, cr, p);
                    r8[qq] = r;
                }
                const uint32_t kr0 = ci * 8;                              // first row within this thread's rows
                const uint32_t nrow = (ch0 + ci) * 8 + 8 <= (uint32_t)RT ? 8u : (uint32_t)RT - (ch0 + ci) * 8;
                // earlier dropped limbs: v <- (v - rho_d) p_{L-1-d}^-1 mod p   (|rho| < p_l / 2 < p)
                if (ndep) {
#pragma unroll
                    for (uint32_t qq = 0; qq < 8; qq++) {
                        const int32_t rh = r8[qq];
                        const uint32_t t = rh < 0 ? addmod(v8[qq], (uint32_t)(-rh), p) : submod(v8[qq], (uint32_t)rh, p);
                        v8[qq] = mulmod_shoup(t, iv_w, iv_sh, p);
                    }
                    for (uint32_t d = 1; d < ndep; d++) {
                        const uint32_t ld = L - 1 - d;
                        const uint32_t w = R.inv_p[ld][limb], wsh = R.inv_p_sh[ld][limb];
                        int32_t rh1[8];
#pragma unroll
                        for (uint32_t qq = 0; qq < 8; qq++)
                            rh1[qq] = qq < nrow ? __ldcg(J.rho + d * rho_stride + ((size_t)(tg0 + kr0 + qq) * 2 + U.comp) * N + Jc)
                                                : 0;
#pragma unroll
                        for (uint32_t qq = 0; qq < 8; qq++) {
                            const int32_t rh = rh1[qq];
                            const uint32_t t = rh < 0 ? addmod(v8[qq], (uint32_t)(-rh), p) : submod(v8[qq], (uint32_t)rh, p);
                            v8[qq] = mulmod_shoup(t, w, wsh, p);
                        }
                    }
                }
                if (!out_pass) {
                    // a dropped limb: keep its centred residues for the later passes
#pragma unroll
                    for (uint32_t qq = 0; qq < 8; qq++)
                        if (qq < nrow)
                            __stcg(J.rho + U.pass * rho_stride + ((size_t)(tg0 + kr0 + qq) * 2 + U.comp) * N + Jc,
                                   v8[qq] > (p >> 1) ? (int32_t)v8[qq] - (int32_t)p : (int32_t)v8[qq]);
                    continue;
                }
                if (masked) {
                    uint32_t rm8[8];
                    const uint64_t zc = z + (uint64_t)kr0 * gN;
#pragma unroll
                    for (uint32_t qq = 0; qq < 8; qq++) {
                        rm8[qq] = (uint32_t)(mix64(zc + qq * gN) >> (64 - R.ell));      // word(seed, 6, tg N + J)
                        v8[qq] = submod(v8[qq], emb_fast(rm8[qq], (uint32_t)R.qout_mod_t, R.ell, p, R.t_inv[limb],
                                                          R.t_inv_sh[limb]), p);
                    }
                    if (r_col) {
#pragma unroll
                        for (uint32_t qq = 0; qq < 8; qq++) {
                            // theta of query qy: row theta R + ri of that query, if it exists
                            const uint32_t thr = th + kr0 + qq, qd = thr / J.nct;
                            const uint32_t th2 = thr - qd * J.nct;
                            if (qq < nrow && tg0 + kr0 + qq < J.ntheta && th2 * J.Rr + ri < J.kq)
                                J.Rout[((size_t)(qy + qd) * J.kq + th2 * J.Rr + ri) * J.n + jj] = rm8[qq];
                        }
                    }
                }
#pragma unroll
                for (uint32_t qq = 0; qq < 8; qq++)
                    if (qq < nrow && tg0 + kr0 + qq < J.ntheta) ctsp[(size_t)(kr0 + qq) * cts_row] = v8[qq];
            }
            PKS_ADD(U.pass < ND ? 13 : 12, t_fin);
            if (U.pass < ND) {
                __threadfence();
                epi_bar();
                if (ew == 0 && lane == 0) st_release(J.flags + U.pass * fl_stride + fl_tile, 1u);
            }
            PKS_ADD(5, t_fin);
            if (U.pass >= ND) PKS_INC(14);
        }
    }
    PKS_FLUSH;
    tc_fence_before();
    if (CL > 1) cluster_sync(); else __syncthreads();   // no CTA leaves while a peer may still multicast into it
    if (warp == 2) {
        tc_fence_after();
        if constexpr (P2) tmem_dealloc2(tmem, 512); else tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ packed X slices
// Item (rc = 2 r + cmp, theta row, kb, 16-byte chunk): row theta_global of theta tile tt
// holds x[q kq + theta R + r] (zero when theta R + r >= kq or theta_global >= ntheta),
// bitwise complemented (S_x bytes) when cmp = 1.
template <int SX, int RT>
__global__ void __launch_bounds__(256) k_slice_pk(const __grid_constant__ PkParams P, uint32_t ell, uint32_t* flag,
                                                  int check, int late) {
    pdl_trigger();
    uint32_t j = 0;
    while (blockIdx.x >= P.job[j].blk_end) j++;
    const PkJob& J = P.job[j];
    const uint32_t idx = (blockIdx.x - (j ? P.job[j - 1].blk_end : 0u)) * blockDim.x + threadIdx.x;
    const uint32_t rows = J.TT * RT;
    const uint32_t per_rc = rows * J.KB * 8;
    const uint32_t rc = idx / per_rc;
    const uint32_t r = rc >> 1, cmp = rc & 1;
    const bool work = rc < 2 * J.Rr && !(r == 0 && cmp);      // term 0 never wraps
    if (late) pdl_wait();         // X is an output of the previous kernel (pdl_outputs_overlap)
    // X (the caller's input) is read and sliced before the PDL wait, while the previous kernel
    // may still run; the counter, the flags and the slices are written after it (the previous
    // contraction may still read them)
    uint32_t w[SX][4];
    size_t base = 0;                 // the operand block of (rc, theta tile, kb)
    uint32_t brow = 0, bc16 = 0;     // the row in the theta tile, the 16-byte chunk
    bool bad = false;
    if (work) {
        const uint32_t rem = idx - rc * per_rc;
        const uint32_t tgl = rem / (J.KB * 8), ch = rem % (J.KB * 8);
        const uint32_t kb = ch >> 3, c16 = ch & 7;
        const uint32_t beta0 = kb * kBK + c16 * 16;
        const uint32_t qy = tgl / J.nct, th = tgl - qy * J.nct;
        const bool present = tgl < J.ntheta && th * J.Rr + r < J.kq;
        const size_t arow = (size_t)qy * J.kq + th * J.Rr + r;
        uint32_t v[16];
        if (present && beta0 + 16 <= J.m && (J.m & 3) == 0) {
            const uint4* src = reinterpret_cast<const uint4*>(J.X + arow * J.m + beta0);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint4 x4 = __ldg(src + q);
                v[4 * q] = x4.x; v[4 * q + 1] = x4.y; v[4 * q + 2] = x4.z; v[4 * q + 3] = x4.w;
            }
        } else {
#pragma unroll
            for (int u = 0; u < 16; u++) v[u] = (present && beta0 + u < J.m) ? J.X[arow * J.m + beta0 + u] : 0u;
        }
        if (check && present && ell < 32) {
            uint32_t any = 0;
#pragma unroll
            for (int u = 0; u < 16; u++) any |= v[u] >> ell;
            bad = any != 0;
        }
        if (cmp) {
            const uint32_t ones = SX >= 4 ? 0xFFFFFFFFu : (1u << (8 * SX)) - 1u;
#pragma unroll
            for (int u = 0; u < 16; u++) v[u] ^= ones;
        }
        const uint32_t tt = tgl / RT, rr = tgl % RT;
#pragma unroll
        for (int i = 0; i < SX; i++)
#pragma unroll
            for (int q = 0; q < 4; q++)
                w[i][q] = ((v[4 * q] >> (8 * i)) & 0xFF) | (((v[4 * q + 1] >> (8 * i)) & 0xFF) << 8) |
                          (((v[4 * q + 2] >> (8 * i)) & 0xFF) << 16) | (((v[4 * q + 3] >> (8 * i)) & 0xFF) << 24);
        // the 128-B swizzle follows the row's position in the whole (S_x x RT)-row operand block:
        // slice i starts at row i RT, which is not a multiple of 8 when RT = 52
        base = ((((size_t)rc * J.TT + tt) * J.KB + kb) * SX * RT) * kBK;
        brow = rr;
        bc16 = c16;
    }
    if (!late) pdl_wait();
    // the contraction's dispatch counter and this job's rho flags start at zero
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.ctr = 0;
    if (idx < J.nflags) J.flags[idx] = 0;
    if (!work) return;
    if (bad) atomicOr(flag, 1u);
#pragma unroll
    for (int i = 0; i < SX; i++)
        *reinterpret_cast<uint4*>(const_cast<uint8_t*>(J.Xp) + base + swz_off(i * RT + brow, bc16)) =
            make_uint4(w[i][0], w[i][1], w[i][2], w[i][3]);
}

// ------------------------------------------------------------------ setup: column sums and corr
// ColSum[col] = sum_{beta < m} E[beta][col] mod p(col), read from the tiled byte planes
// (thread = one coefficient column = one 128-B row of each plane).
__global__ void __launch_bounds__(128) k_colsum(Rns R, const uint8_t* __restrict__ Et, uint32_t KB, uint32_t ncol,
                                                uint32_t* __restrict__ colsum) {
    const uint32_t ct = blockIdx.x, row = threadIdx.x;
    const uint32_t col = ct * kBNW + row;
    if (col >= ncol) return;
    uint32_t sum[kSW] = {0, 0, 0, 0};
    for (uint32_t kb = 0; kb < KB; kb++) {
        const uint8_t* base = Et + ((size_t)ct * KB + kb) * kSW * kBNW * kBK;
#pragma unroll
        for (uint32_t s = 0; s < kSW; s++) {
            const uint4* rp = reinterpret_cast<const uint4*>(base + (size_t)s * kBNW * kBK + row * kBK);
#pragma unroll
            for (int c = 0; c < 8; c++) {          // the 8 chunks of the row, in any (swizzled) order
                const uint4 w = __ldg(rp + c);
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int q = 0; q < 4; q++)
                    sum[s] += (ws[q] & 0xFF) + ((ws[q] >> 8) & 0xFF) + ((ws[q] >> 16) & 0xFF) + (ws[q] >> 24);
            }
        }
    }
    const uint32_t limb = (col / R.N) % R.L, p = R.p[limb];
    uint64_t x = 0;
#pragma unroll
    for (uint32_t s = 0; s < kSW; s++) x += (uint64_t)sum[s] << (8 * s);       // < 2^45
    colsum[col] = reduce64_pm(x, p, R.c32[limb]);
}

// corr[comp][limb][J] = (2^(8 S_x) - 1) sum_{1 <= r < R, J < r n} ColSum[comp][limb][J - r n + N]  mod p
__global__ void k_corr(Rns R, const uint32_t* __restrict__ colsum, uint32_t n, uint32_t SX,
                       uint32_t* __restrict__ corr) {
    const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t N = R.N, ncol = 2 * R.L * N;
    if (col >= ncol) return;
    const uint32_t slab = col / N, J = col % N, limb = slab % R.L, p = R.p[limb];
    const uint32_t Rr = N / n;
    uint64_t s = 0;
    for (uint32_t r = 1; r < Rr; r++)
        if (J < r * n) s += colsum[slab * N + J + N - r * n];
    const uint32_t c = reduce64_pm(s, p, R.c32[limb]);
    // (2^(8 S_x) - 1) mod p: 2^32 - 1 = c32 - 1 (mod p) at S_x = 4
    const uint64_t ones = SX >= 4 ? (uint64_t)R.c32[limb] + p - 1 : (1ull << (8 * SX)) - 1;
    corr[col] = reduce64_pm((uint64_t)c * (ones % p), p, R.c32[limb]);
}

// ------------------------------------------------------------------ host
static uint32_t pk_sx(const nimbus_ctx* c) { return sx_of(c->rns.ell); }

bool packed_layout_ok(const nimbus_ctx* c, const nimbus_encw* w) {
    const char* off = getenv("NIMBUS_NO_PACKED");
    return c->prm.impl == NIMBUS_IMPL_TCGEN05 && w->bn == kBNW && (pk_sx(c) == 4 || pk_sx(c) == 2) &&
           w->n % kBNW == 0 &&
           c->rns.N % kBNW == 0 && c->rns.L - c->rns.L_out >= 1 && c->rns.L - c->rns.L_out <= 2 &&
           !(off && atoi(off) != 0);
}

static uint32_t pk_nct(const nimbus_ctx* c, const nimbus_encw* w, uint32_t kq) {
    const uint32_t Rr = c->rns.N / w->n;
    return (kq + Rr - 1) / Rr;
}

// the packed path pays off once a matmul has enough packed ciphertexts to fill MMA tiles
bool packed_ok(const nimbus_ctx* c, const nimbus_encw* w, uint32_t kq, uint32_t nq) {
    return w->d_corr && w->d_Et && packed_layout_ok(c, w) && nq * pk_nct(c, w, kq) >= 48;
}

// theta-tile heights with an instantiated kernel: S_x = 4 (MMA N = 4 RT <= 256, 7 RT <= 480 TMEM
// columns), S_x = 2 (N = 2 RT, 5 accumulators: RT = 72 fits C5's 208 packed ciphertexts per
// n = 768 matmul in 3 tiles)
static const uint32_t kPkRT4[4] = {48, 52, 56, 64};
static const uint32_t kPkRT2[2] = {64, 72};

// CTA pairs with cta_group::2 MMAs (PkCfg, P2) for a job list -- opt-in, NIMBUS_PK_PAIR=1: S_x = 4,
// every job's shift n / 128 even (the pair's two J tiles then agree on which shift terms wrap, so
// they share the X operand), an even number of J tiles, no NIMBUS_PK_CL.  Measured at C5 (B200,
// sw_power_cap, same box): 90.9-91.3 ms at 1410-1429 MHz vs 90.3 ms at 1444 MHz for the multicast
// pairs (RT = 52 both) -- ~2% fewer cycles per pass, but the pair form reads every Enc(W) plane
// from L2 once per CTA (no theta-tile multicast), and under the board's power cap that energy costs
// the clock the halved smem operand reads win back.
static bool pk_pair_ok(const nimbus_ctx* c, const PkHostJob* jobs, uint32_t count) {
    const char* on = getenv("NIMBUS_PK_PAIR");
    if (!(on && atoi(on) == 1) || getenv("NIMBUS_PK_CL") || pk_sx(c) != 4 || (c->rns.N / kBNW) % 2) return false;
    for (uint32_t j = 0; j < count; j++)
        if ((jobs[j].w->n / kBNW) % 2) return false;
    return count > 0;
}

void packed_rt_candidates(const nimbus_ctx* c, const uint32_t** rts, uint32_t* n) {
    if (pk_sx(c) == 2) { *rts = kPkRT2; *n = 2; } else { *rts = kPkRT4; *n = 4; }
}

// RT minimising the padded MMA work of the job list (ties: the larger RT)
uint32_t packed_rt(const nimbus_ctx* c, const PkHostJob* jobs, uint32_t count) {
    const uint32_t* cand;
    uint32_t ncand;
    packed_rt_candidates(c, &cand, &ncand);
    const char* force = getenv("NIMBUS_PK_RT");       // experiment switch: one of the candidates
    if (force)
        for (uint32_t i = 0; i < ncand; i++)
            if ((uint32_t)atoi(force) == cand[i]) return cand[i];
    uint64_t best = ~0ull;
    uint32_t brt = cand[ncand - 1];
    for (int i = (int)ncand - 1; i >= 0; i--) {
        const uint32_t rt = cand[i];
        uint64_t work = 0;
        for (uint32_t j = 0; j < count; j++) {
            const nimbus_encw* w = jobs[j].w;
            const uint64_t nth = (uint64_t)jobs[j].nq * pk_nct(c, w, jobs[j].kq);
            work += ((nth + rt - 1) / rt) * rt * (c->rns.N / w->n) * w->KB;
        }
        if (work < best) { best = work; brt = rt; }
    }
    return brt;
}

// per job: packed X slices | rho of the dropped limbs | their flags (each 1 KB aligned)
struct PkBytes {
    size_t xp, rho, flags, total;
};
static PkBytes pk_bytes(const nimbus_ctx* c, const nimbus_encw* w, uint64_t ntheta, uint32_t rt) {
    auto al = [](size_t x) { return (x + 1023) & ~size_t(1023); };
    const uint64_t Rr = c->rns.N / w->n, TT = (ntheta + rt - 1) / rt, ND = c->rns.L - c->rns.L_out;
    PkBytes b;
    b.xp = al((size_t)(2 * Rr * TT * w->KB * pk_sx(c) * rt * kBK));
    b.rho = al((size_t)(ND * TT * rt * 2 * c->rns.N * 4));
    b.flags = al((size_t)(ND * 2 * TT * (c->rns.N / kBNW) * 4));
    b.total = b.xp + b.rho + b.flags;
    return b;
}
size_t packed_xp_bytes(const nimbus_ctx* c, const nimbus_encw* w, uint64_t ntheta, uint32_t rt) {
    return pk_bytes(c, w, ntheta, rt).total;
}
size_t packed_job_bytes(const nimbus_ctx* c, const PkHostJob& j, uint32_t rt) {
    return pk_bytes(c, j.w, (uint64_t)j.nq * pk_nct(c, j.w, j.kq), rt).total;
}

// clusters of CL CTAs that can be co-resident (one CTA per SM), cached per kernel
template <typename K>
static uint32_t max_clusters(nimbus_ctx* c, K kernel, uint32_t CL, size_t smem, uint32_t threads) {
    if (CL == 1) return (uint32_t)c->num_sms;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * (c->num_sms / CL));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        return (uint32_t)c->num_sms / CL;
    }
    return (uint32_t)n;
}

// CTAs per cluster of the packed contraction (NIMBUS_PK_CL=1, 2 or 4 overrides): at S_x = 4, 2
// (Enc(W) planes multicast to a theta-tile pair: C5 94.0 vs 95.9 ms single); at S_x = 2, 1 -- each
// plane feeds half the MMA work, and the pair's lockstep costs more than the halved L2 reads (C5@l16:
// 55.0 ms single vs 65.4 paired vs 68.7 in 4-CTA clusters; the MMA warp waited for Enc(W) 20% vs 29%)
static uint32_t pk_cluster(uint32_t sx) {
    const char* e = getenv("NIMBUS_PK_CL");
    const int v = e ? atoi(e) : (sx == 2 ? 1 : 2);
    return v == 1 || v == 4 ? (uint32_t)v : 2u;
}

// unit order within a (pass, component) group: the J tiles walked in shift order with the theta groups
// fastest (pk_decode).  C5 on B200: DRAM reads 39.9 -> 29.8 GB per pass (2.1x -> 1.65x the SURVEY 8(d)
// bytes), 89.1-89.4 -> 88.5-88.7 ms.  NIMBUS_PK_ORDER=0 keeps T fastest (the order before).
static bool pk_walk_order() {
    const char* e = getenv("NIMBUS_PK_ORDER");
    return !e || atoi(e) != 0;
}

template <int SX, int RT, int CL, bool P2 = false>
static cudaError_t launch_pk_rt(nimbus_ctx* c, const PkHostJob* jobs, uint32_t count, uint32_t* d_ctr, cudaStream_t st,
                                void (*mark)(nimbus_ctx*, cudaStream_t)) {
    using Cfg = PkCfg<SX, RT, P2>;
    std::unique_ptr<PkParams> Pp(new PkParams());     // kernel parameters (copied at launch)
    PkParams& P = *Pp;
    c->pf_next = nullptr;                             // a prefetch hint is for a resident-X launch only
    cudaError_t e = ensure_smem(c, k_cop_pk<SX, RT, CL, P2>, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    static uint32_t ncl = 0;                          // one per instantiation
    if (!ncl) ncl = max_clusters(c, k_cop_pk<SX, RT, CL, P2>, CL, Cfg::SMEM, Cfg::THREADS);
    const uint32_t NT = c->rns.N / kBNW, ND = c->rns.L - c->rns.L_out;
    for (uint32_t base = 0; base < count; base += kPkMaxJobs) {
        const uint32_t nj = count - base < kPkMaxJobs ? count - base : kPkMaxJobs;
        memset(&P, 0, sizeof(P));
        P.njobs = nj;
        P.ctr = d_ctr;
        {
            const char* ep = getenv("NIMBUS_PK_EPOL");
            P.epol = ep ? (uint32_t)atoi(ep) : 0u;
#ifdef NIMBUS_PK_DIAG
            const char* dg = getenv("NIMBUS_PK_DIAG");
            P.diag = dg ? (uint32_t)atoi(dg) : 0u;
#endif
        }
        uint32_t units = 0, blocks = 0;
        for (uint32_t i = 0; i < nj; i++) {
            const PkHostJob& h = jobs[base + i];
            PkJob& J = P.job[i];
            const nimbus_encw* w = h.w;
            J.Et = w->d_Et; J.Xp = h.d_Xp; J.corr = w->d_corr; J.cts = h.d_cts; J.Rout = h.d_R; J.X = h.d_X;
            J.key = prg_key(h.seed, 6);
            J.m = w->m; J.KB = w->KB; J.Rr = c->rns.N / w->n; J.n = w->n; J.kq = h.kq;
            J.nct = pk_nct(c, w, h.kq);
            J.ntheta = h.nq * J.nct;
            J.TT = (J.ntheta + RT - 1) / RT;
            J.CKB = kPkMaxChunkKB / J.Rr;
            J.NCH = (J.KB + J.CKB - 1) / J.CKB;
            const PkBytes b = pk_bytes(c, w, J.ntheta, RT);
            J.rho = reinterpret_cast<int32_t*>(const_cast<uint8_t*>(h.d_Xp) + b.xp);
            J.flags = reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(h.d_Xp) + b.xp + b.rho);
            J.nflags = ND * 2 * J.TT * NT;
            if (!P2 && pk_walk_order()) {
                J.ws = (w->n / kBNW) % NT;
                uint32_t a = J.ws, b = NT;
                while (a) { const uint32_t t = b % a; b = a; a = t; }     // b = gcd(ws, NT) (NT if ws = 0)
                J.wc = NT / b;
            }
            units += P2 ? c->rns.L * 2 * J.TT * (NT / 2)               // pair units: J tile pairs
                        : c->rns.L * 2 * ((J.TT + CL - 1) / CL) * NT;  // cluster units: theta tile groups
            J.unit_end = units;
            const uint32_t items = 2 * J.Rr * J.TT * RT * J.KB * 8;
            blocks += ((items > J.nflags ? items : J.nflags) + 255) / 256;
            J.blk_end = blocks;
        }
        const int check = (c->prm.flags & NIMBUS_FLAG_CHECK_RANGE) && c->rns.ell < 32;
        int late = 0;
        for (uint32_t i = 0; i < nj && !late; i++)
            late = pdl_outputs_overlap(st, jobs[base + i].d_X,
                                       (size_t)jobs[base + i].kq * jobs[base + i].nq * jobs[base + i].w->m * 4);
        e = launch_pdl(k_slice_pk<SX, RT>, dim3(blocks), dim3(256), 0, st, P, c->rns.ell, c->d_flag, check, late);
        c->launches++;
        if (e != cudaSuccess) return e;
        if (mark) mark(c, st);
        const uint32_t clusters = units < ncl ? units : ncl;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(clusters * CL);
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
        e = cudaLaunchKernelEx(&cfg, k_cop_pk<SX, RT, CL, P2>, c->rns, P, units);
        c->launches++;
        {   // the contraction writes the jobs' ciphertexts and R, and triggers its dependents early
            std::vector<const void*> op;
            std::vector<size_t> ob;
            for (uint32_t i = 0; i < nj; i++) {
                const PkHostJob& h = jobs[base + i];
                op.push_back(h.d_cts);
                ob.push_back((size_t)h.nq * pk_nct(c, h.w, h.kq) * 2 * c->rns.L_out * c->rns.N * 4);
                op.push_back(h.d_R);
                ob.push_back((size_t)h.kq * h.nq * h.w->n * 4);
            }
            pdl_outputs_set(st, op.data(), ob.data(), (uint32_t)op.size());
        }
        snprintf(c->last_contraction, sizeof(c->last_contraction), P2 ? "k_cop_pk<%d, %d, %d, P2>" : "k_cop_pk<%d, %d, %d>",
                 SX, RT, CL);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <int SX, int RT>
static cudaError_t launch_pk_cl(nimbus_ctx* c, const PkHostJob* jobs, uint32_t count, uint32_t* d_ctr, cudaStream_t st,
                                void (*mark)(nimbus_ctx*, cudaStream_t)) {
    const uint32_t cl = pk_cluster(SX);
    return cl == 2 ? launch_pk_rt<SX, RT, 2>(c, jobs, count, d_ctr, st, mark)
           : cl == 4 ? launch_pk_rt<SX, RT, 4>(c, jobs, count, d_ctr, st, mark)
                     : launch_pk_rt<SX, RT, 1>(c, jobs, count, d_ctr, st, mark);
}

cudaError_t launch_cop_packed(nimbus_ctx* c, const PkHostJob* jobs, uint32_t count, uint32_t rt, uint32_t* d_ctr,
                              cudaStream_t st, void (*mark)(nimbus_ctx*, cudaStream_t)) {
    if (pk_sx(c) == 2) {
        if (rt == 72) return launch_pk_cl<2, 72>(c, jobs, count, d_ctr, st, mark);
        if (rt == 64) return launch_pk_cl<2, 64>(c, jobs, count, d_ctr, st, mark);
        return cudaErrorInvalidValue;
    }
    if (pk_pair_ok(c, jobs, count)) {
        if (rt == 52) return launch_pk_rt<4, 52, 2, true>(c, jobs, count, d_ctr, st, mark);
        if (rt == 56) return launch_pk_rt<4, 56, 2, true>(c, jobs, count, d_ctr, st, mark);
        if (rt == 48) return launch_pk_rt<4, 48, 2, true>(c, jobs, count, d_ctr, st, mark);
        if (rt == 64) return launch_pk_rt<4, 64, 2, true>(c, jobs, count, d_ctr, st, mark);
        return cudaErrorInvalidValue;
    }
    if (rt == 48) return launch_pk_cl<4, 48>(c, jobs, count, d_ctr, st, mark);
    if (rt == 52) return launch_pk_cl<4, 52>(c, jobs, count, d_ctr, st, mark);
    if (rt == 56) return launch_pk_cl<4, 56>(c, jobs, count, d_ctr, st, mark);
    if (rt == 64) return launch_pk_cl<4, 64>(c, jobs, count, d_ctr, st, mark);
    return cudaErrorInvalidValue;
}

// ColSum -> corr for a freshly tiled Enc(W) (every path that fills w->d_Et)
cudaError_t launch_pk_corr(nimbus_ctx* c, nimbus_encw* w, cudaStream_t st) {
    if (!w->d_corr) return cudaSuccess;
    const uint32_t ncol = 2 * c->rns.L * c->rns.N;
    uint32_t* colsum = w->d_corr + ncol;
    k_colsum<<<col_tiles(c, kBNW), 128, 0, st>>>(c->rns, w->d_Et, w->KB, ncol, colsum);
    c->launches++;
    k_corr<<<(ncol + 255) / 256, 256, 0, st>>>(c->rns, colsum, w->n, pk_sx(c), w->d_corr);
    c->launches++;
    return cudaGetLastError();
}

}  // namespace nimbus
