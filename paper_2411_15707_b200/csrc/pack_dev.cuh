// pack_dev.cuh -- device code of K7 (RShift packing + mod-switch + mask), the
// per-item body of k_pack (pack.cu).  See pack.cu for the math and the citations.
#pragma once
#include "internal.h"

namespace nimbus {

// x mod p for a sum of at most 2^13 residues (x < 2^44, rows <= N <= 8192) when c32 = 2^32 mod p < 2^21:
// three folds x = hi 2^32 + lo -> hi c32 + lo (< 3*2^32, < 2^32 + 2^22, < 2^32),
// then two conditional subtractions (2^32 < 3p).
__device__ __forceinline__ uint32_t reduce44_pm(uint64_t x, uint32_t p, uint32_t c32) {
#pragma unroll
    for (int f = 0; f < 3; f++) x = mad_wide((uint32_t)(x >> 32), c32, (uint32_t)x);
    uint32_t r = (uint32_t)x;
    r = r >= p ? r - p : r;
    r = r >= p ? r - p : r;
    return r;
}

template <int V>
struct VecU32;
template <>
struct VecU32<1> {
    __device__ static void load(const uint32_t* p, uint32_t (&v)[1]) { v[0] = __ldg(p); }
    __device__ static void store(uint32_t* p, const uint32_t (&v)[1]) { p[0] = v[0]; }
};
template <>
struct VecU32<2> {
    __device__ static void load(const uint32_t* p, uint32_t (&v)[2]) {
        const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
        v[0] = x.x; v[1] = x.y;
    }
    __device__ static void store(uint32_t* p, const uint32_t (&v)[2]) {
        *reinterpret_cast<uint2*>(p) = make_uint2(v[0], v[1]);
    }
};
template <>
struct VecU32<4> {
    __device__ static void load(const uint32_t* p, uint32_t (&v)[4]) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    }
    __device__ static void store(uint32_t* p, const uint32_t (&v)[4]) {
        *reinterpret_cast<uint4*>(p) = make_uint4(v[0], v[1], v[2], v[3]);
    }
};

// The mask of the work item (component 0 only): r = word(seed, 6, tg N + J + u) >> (64 - ell)
// and Emb_{q'}(r) mod p_i for the output limbs.  It depends on no kernel
// input, so k_pack computes it before its PDL wait, while the contraction still runs.
template <int V, int L, typename MT = uint32_t>
struct PackMask {
    MT r[V];
    uint32_t emb[L][V];
};

template <int V, int L, typename MT = uint32_t>
__device__ __forceinline__ void pack_mask(const Rns& Rn, uint64_t key_mask, uint32_t tg, uint32_t J,
                                          PackMask<V, L, MT>& m) {
    // word(seed, 6, i) = mix64(key + golden (i + 1)) for i = tg N + J + u: one multiply, then steps
    uint64_t z = key_mask + 0x9E3779B97F4A7C15ULL * ((uint64_t)tg * Rn.N + J + 1);
#pragma unroll
    for (int u = 0; u < V; u++, z += 0x9E3779B97F4A7C15ULL) {
        const uint64_t w = mix64(z);
        m.r[u] = (MT)(Rn.ell >= 64 ? w : w >> (64 - Rn.ell));
#pragma unroll
        for (int i = 0; i < L; i++)
            if ((uint32_t)i < Rn.L_out)
                m.emb[i][u] = sizeof(MT) == 8
                                  ? emb_mod(m.r[u], Rn.qout_mod_t, Rn.ell, Rn.p[i], Rn.mu[i], Rn.t_inv[i])
                                  : Rn.ell <= 16
                                  ? emb_fast16((uint32_t)m.r[u], (uint32_t)Rn.qout_mod_t, Rn.ell, Rn.p[i],
                                               Rn.t_inv[i], Rn.t_inv_sh[i])
                                  : emb_fast((uint32_t)m.r[u], (uint32_t)Rn.qout_mod_t, Rn.ell, Rn.p[i],
                                             Rn.t_inv[i], Rn.t_inv_sh[i]);
    }
}

// One work item of K7: coefficients J..J+V-1 of component `comp` of packed
// ciphertext tg (all limbs).  RB rows of loads are in flight per batch; the host
// picks RB to fit R = floor(N/n) (1 for C3, 5 for C2, ...) so that few load slots
// are predicated off -- the kernel is issue-bound, not bandwidth-bound.
// MT: element type of the mask / R (uint64_t for ell > 32, then V = 1).
template <int V, int L, int RB, typename MT = uint32_t>
__device__ __forceinline__ void pack_item(const Rns& Rn, const uint32_t* __restrict__ C, uint32_t kq, uint32_t n,
                                          uint32_t Rr, uint32_t nct, uint64_t key_mask, uint32_t* __restrict__ cts,
                                          MT* __restrict__ Rout, const uint32_t* __restrict__ Z0, uint32_t tg,
                                          uint32_t comp, uint32_t J, const PackMask<V, L, MT>& mk) {
    static_assert(sizeof(MT) == 4 || V == 1, "64-bit masks: one coefficient per thread");
    const uint32_t N = Rn.N, Lo = Rn.L_out;
    const uint32_t query = tg / nct, theta = tg - query * nct;
    const uint32_t rows = min(Rr, kq - theta * Rr);
    const uint32_t ncol = 2u * L * N;          // row offsets below stay in 32 bits (rows * ncol < 2^30)
    const size_t row0 = (size_t)query * kq + (size_t)theta * Rr;
    const uint32_t* Cq = C + row0 * ncol + comp * L * N;

    uint64_t acc[L][V];
#pragma unroll
    for (int i = 0; i < L; i++)
#pragma unroll
        for (int u = 0; u < V; u++) acc[i][u] = 0;
#pragma unroll 1
    for (uint32_t r0 = 0; r0 < rows; r0 += RB) {
        uint32_t v[RB][L][V];
        bool wrap[RB];
#pragma unroll
        for (int b = 0; b < RB; b++) {
            const uint32_t r = r0 + b, s = r * n;
            wrap[b] = J < s;
            const uint32_t idx = wrap[b] ? J + N - s : J - s;
#pragma unroll
            for (int i = 0; i < L; i++) {
                if (r < rows) {
                    VecU32<V>::load(Cq + (r * ncol + i * N + idx), v[b][i]);
                } else {
#pragma unroll
                    for (int u = 0; u < V; u++) v[b][i][u] = 0;
                }
            }
        }
#pragma unroll
        for (int b = 0; b < RB; b++) {
            if (r0 + b < rows) {
#pragma unroll
                for (int i = 0; i < L; i++)
#pragma unroll
                    for (int u = 0; u < V; u++) acc[i][u] += wrap[b] ? Rn.p[i] - v[b][i][u] : v[b][i][u];
            }
        }
    }
    if (Z0) {
        // circuit privacy: + Enc_pk(0) at the full modulus, before the mod-switch (reading 26)
#pragma unroll
        for (int i = 0; i < L; i++) {
            uint32_t z[V];
            VecU32<V>::load(Z0 + (((size_t)tg * 2 + comp) * L + i) * N + J, z);
#pragma unroll
            for (int u = 0; u < V; u++) acc[i][u] += z[u];
        }
    }
    uint32_t out[L][V];
#pragma unroll
    for (int u = 0; u < V; u++) {
        uint32_t res[L];
#pragma unroll
        for (int i = 0; i < L; i++) {
            // RB == 1: a single unwrapped row (R = 1) plus at most one zero-encryption residue (< 2 p)
            if (RB == 1) {
                const uint32_t r = (uint32_t)acc[i][u];
                res[i] = r >= Rn.p[i] ? r - Rn.p[i] : r;
            } else {
                res[i] = reduce44_pm(acc[i][u], Rn.p[i], Rn.c32[i]);
            }
        }
#pragma unroll
        for (int l = L - 1; l >= 1; l--) {
            if ((uint32_t)l >= Lo) {
                const uint32_t pl = Rn.p[l], c = res[l];
                const bool neg = c > (pl >> 1);          // centered rho = c - p_l < 0
                const uint32_t mag = neg ? pl - c : c;   // |rho| < p_l / 2 < p_i
#pragma unroll
                for (int i = 0; i < l; i++) {
                    const uint32_t p = Rn.p[i];
                    const uint32_t d = neg ? addmod(res[i], mag, p) : submod(res[i], mag, p);
                    res[i] = mulmod_shoup(d, Rn.inv_p[l][i], Rn.inv_p_sh[l][i], p);
                }
            }
        }
        if (comp == 0) {
#pragma unroll
            for (int i = 0; i < L; i++)
                if ((uint32_t)i < Lo) res[i] = submod(res[i], mk.emb[i][u], Rn.p[i]);
        }
#pragma unroll
        for (int i = 0; i < L; i++) out[i][u] = res[i];
    }
#pragma unroll
    for (int i = 0; i < L; i++)
        if ((uint32_t)i < Lo) VecU32<V>::store(cts + (((size_t)tg * 2 + comp) * Lo + i) * N + J, out[i]);
    if (comp == 0 && Rout && J < rows * n) {          // Rout null: R written by k_mask_R instead
        if (sizeof(MT) == 8) Rout[row0 * n + J] = mk.r[0];
        else VecU32<V>::store(reinterpret_cast<uint32_t*>(Rout) + row0 * n + J,
                              reinterpret_cast<const uint32_t(&)[V]>(mk.r));
    }
}

}  // namespace nimbus
