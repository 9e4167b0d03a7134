// common.cuh -- device helpers shared by the Nimbus COP kernels (sm_100a).
// PRG contract, modular arithmetic, and the raw PTX
// wrappers for mbarrier / bulk async copy / tcgen05 used by the contraction.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define NIMBUS_MAXL 6

namespace nimbus {

// ------------------------------------------------------------------ constants
// Per-context RNS constants, passed to kernels by value.
struct Rns {
    uint32_t N, logN, L, L_out, ell;
    uint32_t p[NIMBUS_MAXL];
    uint64_t mu[NIMBUS_MAXL];            // floor(2^64 / p_i)            (Barrett)
    uint32_t inv_p[NIMBUS_MAXL][NIMBUS_MAXL];  // inv_p[l][i] = p_l^-1 mod p_i (mod-switch)
    uint32_t inv_p_sh[NIMBUS_MAXL][NIMBUS_MAXL];  // Shoup companions floor(inv_p * 2^32 / p_i)
    uint32_t t_inv[NIMBUS_MAXL];         // t^-1 mod p_i                 (embedding)
    uint32_t t_inv_sh[NIMBUS_MAXL];      // floor(t_inv * 2^32 / p_i)
    uint64_t q_mod_t;                    // q mod t, q = prod of all L primes (t = 2^ell <= 2^64)
    uint64_t qout_mod_t;                 // q' mod t, q' = prod of the first L_out primes
    uint32_t pow8[NIMBUS_MAXL][12];      // 2^(8s) mod p_i, s < S_x + 3   (slice recombination)
    uint32_t c32[NIMBUS_MAXL];           // 2^32 mod p_i (< 2^21 required by reduce64_pm)
    uint32_t ninv[NIMBUS_MAXL], ninv_sh[NIMBUS_MAXL];  // N^-1 mod p_i and its Shoup companion
};

// ------------------------------------------------------------------ PRG
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}
__host__ __device__ __forceinline__ uint64_t prg_key(uint64_t seed, uint32_t dom) {
    return mix64(seed ^ ((uint64_t)dom << 56));
}
// word(seed, dom, i) with the key precomputed
__host__ __device__ __forceinline__ uint64_t prg_word(uint64_t key, uint64_t i) {
    return mix64(key + 0x9E3779B97F4A7C15ULL * (i + 1));
}
__device__ __forceinline__ uint32_t samp_uniform_mod(uint64_t w, uint32_t p) {
    return (uint32_t)__umul64hi(w, (uint64_t)p);
}
__device__ __forceinline__ int32_t samp_ternary(uint64_t w) {
    return (int32_t)__umul64hi(w, 3ULL) - 1;
}
__device__ __forceinline__ int32_t samp_cbd21(uint64_t w) {
    return __popcll(w & 0x1FFFFFULL) - __popcll((w >> 21) & 0x1FFFFFULL);
}
__device__ __forceinline__ uint32_t samp_mod_t(uint64_t w, uint32_t ell) {
    return (uint32_t)(w >> (64 - ell));
}

// ------------------------------------------------------------------ modular
// x mod p for any 64-bit x (Barrett with mu = floor(2^64/p): q_hat <= x/p < q_hat + 2)
__device__ __forceinline__ uint32_t mod64(uint64_t x, uint32_t p, uint64_t mu) {
    uint64_t qh = __umul64hi(x, mu);
    uint64_t r = x - qh * (uint64_t)p;
    return (uint32_t)(r >= p ? r - p : r);
}
__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t b, uint32_t p, uint64_t mu) {
    return mod64((uint64_t)a * b, p, mu);
}
__device__ __forceinline__ uint32_t addmod(uint32_t a, uint32_t b, uint32_t p) {
    uint32_t s = a + b;   // a, b < p < 2^31: no overflow
    return s >= p ? s - p : s;
}
__device__ __forceinline__ uint32_t submod(uint32_t a, uint32_t b, uint32_t p) {
    return a >= b ? a - b : a + p - b;
}
// Shoup: w_sh = floor(w * 2^32 / p); returns a*w mod p for a < 2^32
__device__ __forceinline__ uint32_t mulmod_shoup(uint32_t a, uint32_t w, uint32_t w_sh, uint32_t p) {
    uint32_t q = __umulhi(a, w_sh);
    uint32_t r = a * w - q * p;
    return r >= p ? r - p : r;
}

// a * b + c with a 32x32 -> 64-bit multiply-add (one IMAD.WIDE.U32)
__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) { return (uint64_t)a * b + c; }

// x mod p for any 64-bit x when c32 = 2^32 mod p < 2^21 (true for the primes
// within 2^20 of 2^31 that the context derives): fold x = hi 2^32 + lo ->
// hi c32 + lo three times (< 2^53 + 2^32, < 2^42 + 2^33, < 2^32 + 2^31 + 2^21),
// then the last carry h in {0, 1} as h c32 on the low word (l < 2^31 + 2^21 when
// h = 1, so the sum stays below 2^32 < 3p), then at most two conditional
// subtractions.  Three IMAD.WIDE instead of five: the epilogue that calls it per
// output is bound by the FMA pipe.
__device__ __forceinline__ uint32_t reduce64_pm(uint64_t x, uint32_t p, uint32_t c32) {
#pragma unroll
    for (int f = 0; f < 3; f++) x = mad_wide((uint32_t)(x >> 32), c32, (uint32_t)x);
    uint32_t r = (uint32_t)x + ((uint32_t)(x >> 32) ? c32 : 0u);
    r = r >= p ? r - p : r;
    r = r >= p ? r - p : r;
    return r;
}

// Emb(w) mod p_i for w in [0,t): floor((Q w + t/2)/t) = (Q w + t/2 - f)/t with
// f = (Q w + t/2) mod t; since p_i | Q this is (t/2 - f) * t^-1 mod p_i.
// (SURVEY.md §8(c) #4.)  qmodt = Q mod t.  All arithmetic mod 2^64, so ell = 64
// (the paper's t) is the same formula with the mask omitted.
__device__ __forceinline__ uint32_t emb_mod(uint64_t w, uint64_t qmodt, uint32_t ell, uint32_t p,
                                            uint64_t mu, uint32_t tinv) {
    const uint64_t half = 1ULL << (ell - 1);
    const uint64_t tmask = ell >= 64 ? ~0ULL : (half << 1) - 1;
    const uint64_t f = (qmodt * w + half) & tmask;
    // (t/2 - f) mod p, |t/2 - f| <= t/2
    const uint32_t dr = f <= half ? mod64(half - f, p, mu) : (p - mod64(f - half, p, mu)) % p;
    return mulmod(dr, tinv, p, mu);
}

// Emb_{Q}(w) mod p with 32-bit Shoup multiplication:
// (t/2 - f) * t^-1 mod p,  f = (Q w + t/2) mod t,  |t/2 - f| <= t/2 < 2p.
__device__ __forceinline__ uint32_t emb_fast(uint32_t w, uint32_t qmodt, uint32_t ell, uint32_t p, uint32_t tinv,
                                             uint32_t tinv_sh) {
    const uint64_t t = 1ULL << ell;
    const uint64_t f = ((uint64_t)qmodt * w + (t >> 1)) & (t - 1);
    int64_t d = (int64_t)(t >> 1) - (int64_t)f;
    if (d < 0) d += p;
    if (d < 0) d += p;
    if (d >= (int64_t)p) d -= p;
    return mulmod_shoup((uint32_t)d, tinv, tinv_sh, p);
}

// Emb_{Q}(w) mod p for ell <= 16, all in 32 bits: Q w + t/2 < 2^32 when Q < t = 2^ell.
__device__ __forceinline__ uint32_t emb_fast16(uint32_t w, uint32_t qmodt, uint32_t ell, uint32_t p, uint32_t tinv,
                                               uint32_t tinv_sh) {
    const uint32_t t = 1u << ell;
    const uint32_t f = (qmodt * w + (t >> 1)) & (t - 1);
    const uint32_t h = t >> 1;
    const uint32_t d = h >= f ? h - f : p - (f - h);     // (t/2 - f) mod p, |t/2 - f| <= t/2 < p
    return mulmod_shoup(d, tinv, tinv_sh, p);
}

// ------------------------------------------------------------------ PTX: mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}"
        :: "r"(smem_u32(bar)), "r"(parity), "r"(0x989680) : "memory");
}

// ------------------------------------------------------------------ PTX: bulk copy
// 1-D bulk async copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;"
        :: "r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// Same, multicast to every CTA of the cluster in cta_mask (same smem offset, and
// complete_tx on the mbarrier at the same offset in each destination CTA).
__device__ __forceinline__ void bulk_g2s_mc(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                            uint32_t cta_mask, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4, %5;"
        :: "r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "h"((uint16_t)cta_mask),
           "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Bulk prefetch of [p, p + bytes) into L2 (no shared memory, no completion tracking).
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" :: "l"(p), "r"(bytes), "l"(pol) : "memory");
}

// ------------------------------------------------------------------ PDL
// Programmatic dependent launch: wait for the preceding kernel of the stream
// (complete, memory visible) / allow the next one to be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------ PTX: tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(dst_smem)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::i8 (u8 x u8 -> s32)
__device__ __forceinline__ void mma_i8_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// Warp-converged variants: the whole warp executes the call with identical (warp-uniform)
// operands and one lane, chosen by elect.sync inside the asm, issues the instruction.  With
// the issue under `if (lane == 0)` the compiler cannot prove the operands uniform and wraps
// every tcgen05.mma in an ELECT / R2UR.BROADCAST / BRA.U.ANY loop (~25 instructions per MMA,
// more than a 104-cycle MMA leaves for its issue).
__device__ __forceinline__ void mma_i8_ss_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem], kind::i8, warp-converged
__device__ __forceinline__ void mma_i8_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
        :: "r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void mma_commit_mc_w(uint64_t* bar, uint32_t cta_mask) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
        :: "r"(smem_u32(bar)), "h"((uint16_t)cta_mask) : "memory");
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
        :: "r"(smem_u32(bar)) : "memory");
}

// arrive on an mbarrier when all prior tcgen05.mma of this thread complete
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}
// arrive on the mbarrier at this offset in every CTA of cta_mask when all prior MMAs complete
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint32_t cta_mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"((uint16_t)cta_mask) : "memory");
}
// 32 lanes x 32b, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor, K-major, 128-byte swizzle: rows of 128 B,
// 8-row swizzle atoms of 1024 B stacked along M/N (SBO = 1024), version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc_kmajor_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);         // start address
    d |= (uint64_t)(0) << 16;                            // LBO (unused for swizzled K-major)
    d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;         // SBO
    d |= (uint64_t)1 << 46;                              // version = 1
    d |= (uint64_t)2 << 61;                              // SWIZZLE_128B
    return d;
}
// Instruction descriptor kind::i8: D=s32, A=u8, B=u8, both K-major.
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
    return (2u << 4)            // c_format = S32
         | (0u << 7)            // a_format = unsigned 8-bit
         | (0u << 10)           // b_format = unsigned 8-bit
         | ((N >> 3) << 17)     // n_dim
         | ((M >> 4) << 24);    // m_dim
}

}  // namespace nimbus
