// encrypt.cu -- K3, Encrypt rows (Alg. 1 step 1) fused end to
// end: sample a, NTT(a), (.) s_hat, iNTT, + Emb_q(w_hat) + e, and the write of both components
// straight into the contraction's byte-plane layout (layout.cu) -- no canonical intermediate.
//
// Per (row beta, limb i):   a     = uniform mod p_i             (domain 2, index (beta L + i) N + j)
//                           b     = a s + Emb_q(w_hat) + e mod p_i  (e: CBD(21), domain 3, index beta N + j)
//                           w_hat = W[beta][j] for j < n, else 0    (Eq. 2)
// -- the same definition as the two-pass k_encrypt + k_tile_encw (ntt.cu, layout.cu), which stay
// for ring degrees other than 4096 / 8192.
//
// Shape.  One CTA per (beta, limb) with T = N / 16 threads, 16 residues per thread in registers.
// A pass runs 4 butterfly stages on a thread's 16 residues (radix 16); passes exchange through
// shared memory (ping-pong: one barrier per pass), XOR-swizzled per ring degree so that every
// pass's warp access is bank-conflict free.  At N = 8192 the 13th stage (t = 1) pairs lanes
// 2i, 2i+1 and is a warp-shuffle stage.  The pointwise product with s_hat sits between the
// forward's last and the inverse's first register pass (no shared-memory round trip); s_hat
// comes pre-permuted into that pass's thread order with its Shoup companions (k_perm_s, at
// KeyGen).  Forward: Cooley-Tukey, natural -> bit-reversed; inverse: Gentleman-Sande back, the
// N^-1 scaling folded into the epilogue: the same transforms as ntt.cu, regrouped.
//
// Transpose.  A cluster of kEncRows = 8 CTAs holds 8 consecutive rows = half a 16-byte chunk of
// each 128-byte plane row.  After the cluster barrier, CTA rank c gathers coefficient columns
// [c N/8, (c+1) N/8) of the 8 rows from its peers' shared memory (two columns per thread) and
// stores, per component and column, 4 planes x 8 bytes; the neighbouring cluster, running at the
// same time, fills the chunk's other half in L2.  HBM traffic is the bytes written (2 L N 4 per
// row) plus W.
#include "ntt_dev.cuh"
#include "slice_dev.cuh"

namespace nimbus {

#ifndef NIMBUS_ENC_ROWS
#define NIMBUS_ENC_ROWS 8
#endif
// rows per cluster (8: half a 16-B chunk of a 128-B plane row; 16: a whole chunk).  16-CTA clusters
// (non-portable) fit only 14 at once on the B200's GPCs -- 112 of 148 SMs busy
constexpr uint32_t kEncRows = NIMBUS_ENC_ROWS;

template <int LOGN>
struct EncGeo {
    static constexpr uint32_t N = 1u << LOGN, T = N / 16;
    static constexpr uint32_t S1 = N / 256, S2 = N / 4096;   // residue strides of passes 1, 2 (pass 0: T)
};

// Shared-memory word of coefficient w: the 5 bank bits XOR a function of the 32-word row w >> 5.
// Pass accesses (per warp, one k): pass 0 / N=8192 pass 1 -- 32 consecutive words of one row;
// N=8192 pass 2 -- rows b..b+15 x offsets {2k, 2k+1}: (row & 15) << 1 spreads them over all 32
// banks; N=4096 pass 1 -- rows r, r+8 x 16 offsets: bit 4 must differ, so bit 3 of the row goes
// to bank bit 4; N=4096 pass 2 -- rows r..r+15 x offsets {k, 16+k}: the low 4 bits take row & 15.
template <int LOGN>
__device__ __forceinline__ uint32_t enc_pos(uint32_t w) {
    const uint32_t row = w >> 5;
    return w ^ (LOGN == 13 ? (row & 15u) << 1 : (row & 15u) | ((row & 8u) << 1));
}

// residue k of thread g in a pass whose groups are 16 residues at stride S
template <uint32_t S>
__device__ __forceinline__ uint32_t pass_idx(uint32_t g, uint32_t k) {
    return (g / S) * 16 * S + g % S + S * k;
}
template <int LOGN, uint32_t S>
__device__ __forceinline__ void pass_ld(const uint32_t* s, uint32_t (&x)[16], uint32_t g) {
#pragma unroll
    for (uint32_t k = 0; k < 16; k++) x[k] = s[enc_pos<LOGN>(pass_idx<S>(g, k))];
}
template <int LOGN, uint32_t S>
__device__ __forceinline__ void pass_st(uint32_t* s, const uint32_t (&x)[16], uint32_t g) {
#pragma unroll
    for (uint32_t k = 0; k < 16; k++) s[enc_pos<LOGN>(pass_idx<S>(g, k))] = x[k];
}

// Lazy butterflies: values travel in [0, 2p) (p < 2^31, so 2p < 2^32) and each butterfly reduces
// only what its sums need: x and S y to [0, p) by one subtract + unsigned min, the products left
// in Shoup's [0, 2p).  9 integer instructions instead of 11-12, 3 of them on the ALU pipe instead
// of 7.  The pointwise product and the N^-1 scaling are full Shoup reductions, so the values that
// leave the transform are in [0, p).
__device__ __forceinline__ uint32_t red2(uint32_t x, uint32_t p) { return min(x, x - p); }   // [0,2p) -> [0,p)
__device__ __forceinline__ uint32_t shoup_lazy(uint32_t a, uint32_t w, uint32_t w_sh, uint32_t p) {
    return a * w - __umulhi(a, w_sh) * p;                                                     // [0, 2p)
}
__device__ __forceinline__ void ct_lazy(uint32_t& x, uint32_t& y, uint32_t S, uint32_t Ssh, uint32_t p) {
    const uint32_t xr = red2(x, p), V = red2(shoup_lazy(y, S, Ssh, p), p);
    x = xr + V;
    y = xr - V + p;
}
__device__ __forceinline__ void gs_lazy(uint32_t& x, uint32_t& y, uint32_t S, uint32_t Ssh, uint32_t p) {
    const uint32_t xr = red2(x, p), yr = red2(y, p);
    x = xr + yr;
    y = shoup_lazy(xr - yr + p, S, Ssh, p);
}

// 4 forward stages from stage s0 (m0 = 2^s0 blocks of N >> s0) on the thread's block blk:
// stage q pairs residues k, k + 8 >> q; block index (m0 + blk) 2^q + (k >> (4 - q)).
__device__ __forceinline__ void fwd_pass(uint32_t (&x)[16], uint32_t m0, uint32_t blk, const uint32_t* tw,
                                         const uint32_t* tw_sh, uint32_t p) {
#pragma unroll
    for (uint32_t q = 0; q < 4; q++) {
        const uint32_t half = 8u >> q;
#pragma unroll
        for (uint32_t sub = 0; sub < (1u << q); sub++) {
            const uint32_t ti = ((m0 + blk) << q) + sub;
            const uint32_t S = __ldg(tw + ti), Ssh = __ldg(tw_sh + ti);
#pragma unroll
            for (uint32_t kk = 0; kk < half; kk++) ct_lazy(x[sub * 2 * half + kk], x[sub * 2 * half + kk + half], S, Ssh, p);
        }
    }
}
// 4 inverse stages t = S, 2S, 4S, 8S (h0 = N / 2S blocks at the first): stage q pairs residues
// k, k + 2^q; block index (h0 >> q) + blk (8 >> q) + (k >> (q + 1)).
__device__ __forceinline__ void inv_pass(uint32_t (&x)[16], uint32_t h0, uint32_t blk, const uint32_t* iv,
                                         const uint32_t* iv_sh, uint32_t p) {
#pragma unroll
    for (uint32_t q = 0; q < 4; q++) {
        const uint32_t dist = 1u << q, nsub = 8u >> q;
#pragma unroll
        for (uint32_t sub = 0; sub < nsub; sub++) {
            const uint32_t ti = (h0 >> q) + blk * nsub + sub;
            const uint32_t S = __ldg(iv + ti), Ssh = __ldg(iv_sh + ti);
#pragma unroll
            for (uint32_t kk = 0; kk < dist; kk++) gs_lazy(x[sub * 2 * dist + kk], x[sub * 2 * dist + kk + dist], S, Ssh, p);
        }
    }
}
// 16 consecutive table words t[0..15] (16-byte aligned) as four 128-bit loads
__device__ __forceinline__ void ld16(const uint32_t* t, uint32_t (&v)[16]) {
#pragma unroll
    for (uint32_t u = 0; u < 4; u++) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(t) + u);
        v[4 * u] = q.x; v[4 * u + 1] = q.y; v[4 * u + 2] = q.z; v[4 * u + 3] = q.w;
    }
}

// plane s (byte s) of 4 residues: (w0.s, w1.s, w2.s, w3.s)
__device__ __forceinline__ void planes4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&pl)[4]) {
    const uint32_t lo01 = __byte_perm(w0, w1, 0x5140), lo23 = __byte_perm(w2, w3, 0x5140);
    const uint32_t hi01 = __byte_perm(w0, w1, 0x7362), hi23 = __byte_perm(w2, w3, 0x7362);
    pl[0] = __byte_perm(lo01, lo23, 0x5410);
    pl[1] = __byte_perm(lo01, lo23, 0x7632);
    pl[2] = __byte_perm(hi01, hi23, 0x5410);
    pl[3] = __byte_perm(hi01, hi23, 0x7632);
}

template <int LOGN, typename TW>
__global__ void __launch_bounds__(EncGeo<LOGN>::T, 2)
k_encrypt_planes(Rns R, const uint32_t* __restrict__ d_tw, const uint32_t* __restrict__ s_enc,
                 const TW* __restrict__ W, uint32_t m, uint32_t n, uint64_t seed, uint32_t KB, uint32_t bn,
                 uint8_t* __restrict__ Et) {
    using G = EncGeo<LOGN>;
    constexpr uint32_t N = G::N, T = G::T, S1 = G::S1, S2 = G::S2;
    constexpr uint64_t GOLD = 0x9E3779B97F4A7C15ULL;
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* sA = sm;              // a, natural order (the gather's component 1)
    uint32_t* sP = sm + N;          // ping (and b, natural order, at the end)
    uint32_t* sQ = sm + 2 * N;      // pong
    const uint32_t g = threadIdx.x, beta = blockIdx.x, i = blockIdx.y, L = R.L, p = R.p[i];
    if (beta < m) {
        const uint32_t* tw = d_tw + (size_t)i * 4 * N;
        const uint32_t *fw = tw, *fw_sh = tw + N, *iv = tw + 2 * N, *iv_sh = tw + 3 * N;
        uint32_t x[16];
        // a: residue j = g + T k (pass-0 order), PRG counter stepped by T
        uint64_t za = prg_key(seed, 2) + GOLD * (((uint64_t)beta * L + i) * N + g + 1);
#pragma unroll
        for (uint32_t k = 0; k < 16; k++, za += GOLD * T) {
            x[k] = samp_uniform_mod(mix64(za), p);
            sA[enc_pos<LOGN>(g + T * k)] = x[k];
        }
        // ---- forward NTT(a): stages t = N/2 .. N/32 | N/64 .. N/512 | N/1024 .. N/8192 (+ t = 1 at 8192)
        fwd_pass(x, 1, 0, fw, fw_sh, p);
        pass_st<LOGN, T>(sP, x, g);
        __syncthreads();
        pass_ld<LOGN, S1>(sP, x, g);
        fwd_pass(x, 16, g / S1, fw, fw_sh, p);
        pass_st<LOGN, S1>(sQ, x, g);
        __syncthreads();
        pass_ld<LOGN, S2>(sQ, x, g);
        fwd_pass(x, 256, g / S2, fw, fw_sh, p);
        const uint32_t blk2 = g / S2, jj = g % S2;         // at N = 8192: the lane pair (2i, 2i+1) = jj
        if (LOGN == 13) {
            // stage t = 1: residues blk2 32 + 2k (jj = 0) and + 1 (jj = 1), block blk2 16 + k
            uint32_t S[16], Ssh[16];
            ld16(fw + N / 2 + blk2 * 16, S);
            ld16(fw_sh + N / 2 + blk2 * 16, Ssh);
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) {
                const uint32_t o = __shfl_xor_sync(0xffffffffu, x[k], 1);
                const uint32_t V = red2(shoup_lazy(jj ? x[k] : o, S[k], Ssh[k], p), p);
                const uint32_t xe = red2(jj ? o : x[k], p);                // the even residue, reduced
                x[k] = jj ? xe - V + p : xe + V;
            }
        }
        {   // (.) s_hat, in this pass's thread order
            uint32_t sv[16], ssh[16];
            ld16(s_enc + (size_t)i * N + g * 16, sv);
            ld16(s_enc + (size_t)(L + i) * N + g * 16, ssh);
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) x[k] = mulmod_shoup(x[k], sv[k], ssh[k], p);
        }
        // ---- inverse NTT: (t = 1 at 8192) | S2 .. 8 S2 | S1 .. 8 S1 | T .. 8 T
        if (LOGN == 13) {
            uint32_t S[16], Ssh[16];
            ld16(iv + N / 2 + blk2 * 16, S);
            ld16(iv_sh + N / 2 + blk2 * 16, Ssh);
#pragma unroll
            for (uint32_t k = 0; k < 16; k++) {
                const uint32_t o = red2(__shfl_xor_sync(0xffffffffu, x[k], 1), p), v = red2(x[k], p);
                x[k] = jj ? shoup_lazy(o - v + p, S[k], Ssh[k], p) : v + o;
            }
        }
        inv_pass(x, N / (2 * S2), blk2, iv, iv_sh, p);
        pass_st<LOGN, S2>(sP, x, g);
        __syncthreads();
        pass_ld<LOGN, S1>(sP, x, g);
        inv_pass(x, N / (2 * S1), g / S1, iv, iv_sh, p);
        pass_st<LOGN, S1>(sQ, x, g);
        __syncthreads();
        pass_ld<LOGN, T>(sQ, x, g);
        inv_pass(x, 8, 0, iv, iv_sh, p);
        // ---- b = N^-1 iNTT(.) + Emb_q(w_hat) + e  at j = g + T k
        uint64_t ze = prg_key(seed, 3) + GOLD * ((uint64_t)beta * N + g + 1);
        const uint32_t ninv = R.ninv[i], ninv_sh = R.ninv_sh[i];
#pragma unroll
        for (uint32_t k = 0; k < 16; k++, ze += GOLD * T) {
            const uint32_t j = g + T * k;
            const uint32_t as = mulmod_shoup(x[k], ninv, ninv_sh, p);
            const uint64_t w = j < n ? (uint64_t)W[(size_t)beta * n + j] : 0u;
            const int32_t e = samp_cbd21(mix64(ze));
            const uint32_t em = R.ell > 32 ? emb_mod(w, R.q_mod_t, R.ell, p, R.mu[i], R.t_inv[i])
                                : R.ell <= 16 ? emb_fast16((uint32_t)w, (uint32_t)R.q_mod_t, R.ell, p, R.t_inv[i], R.t_inv_sh[i])
                                              : emb_fast((uint32_t)w, (uint32_t)R.q_mod_t, R.ell, p, R.t_inv[i], R.t_inv_sh[i]);
            const uint32_t er = e < 0 ? p - (uint32_t)(-e) : (uint32_t)e;
            sP[enc_pos<LOGN>(j)] = addmod(addmod(as, em, p), er, p);
        }
    } else {
        // rows m .. KB 128: zero planes (the contraction reads whole 128-row k-blocks)
#pragma unroll
        for (uint32_t k = 0; k < 16; k++) {
            sA[enc_pos<LOGN>(g + T * k)] = 0;
            sP[enc_pos<LOGN>(g + T * k)] = 0;
        }
    }
    cluster_sync();     // the cluster's rows' (b, a) are in their CTAs' shared memory
    // ---- transpose: column j of the cluster's kEncRows rows -> 4 planes x kEncRows bytes per component
    constexpr uint32_t ROWS = kEncRows, CPT = 16 / ROWS;      // columns per thread
    const uint32_t rank = cluster_ctarank();
    const uint32_t beta0 = blockIdx.x & ~(ROWS - 1), kb = beta0 / kBK;
    const uint32_t c16 = (beta0 % kBK) / 16, b16 = beta0 % 16;  // 16-B chunk of the plane row, byte within
#pragma unroll
    for (uint32_t cc = 0; cc < CPT; cc++) {
        const uint32_t j = (rank * CPT + cc) * T + g;
#pragma unroll
        for (uint32_t comp = 0; comp < 2; comp++) {
            const uint32_t* buf = comp ? sA : sP;
            uint32_t w[ROWS];
#pragma unroll
            for (uint32_t q = 0; q < ROWS; q++) w[q] = ld_dsmem(dsmem_addr(buf + enc_pos<LOGN>(j), q));
            uint32_t pl[4][ROWS / 4];
#pragma unroll
            for (uint32_t u = 0; u < ROWS / 4; u++) {
                uint32_t t4[4];
                planes4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3], t4);
#pragma unroll
                for (uint32_t s = 0; s < 4; s++) pl[s][u] = t4[s];
            }
            const uint32_t col = (comp * L + i) * N + j, ct = col / bn, r = col - ct * bn;
            uint8_t* base = Et + ((size_t)ct * KB + kb) * kSW * bn * kBK + swz_off(r, c16) + b16;
#pragma unroll
            for (uint32_t s = 0; s < 4; s++) {
                if constexpr (ROWS == 16)
                    *reinterpret_cast<uint4*>(base + (size_t)s * bn * kBK) = make_uint4(pl[s][0], pl[s][1], pl[s][2], pl[s][3]);
                else
                    *reinterpret_cast<uint2*>(base + (size_t)s * bn * kBK) = make_uint2(pl[s][0], pl[s][1]);
            }
        }
    }
    // no CTA leaves while a peer may still read its shared memory.  Relaxed arrive: the gathered
    // values were consumed (stored) before it, and a release would wait for those global stores
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

// s_hat (bit-reversed NTT order, KeyGen) -> the order of the last forward pass's threads:
// s_enc[i][g][k] = s_hat_i[pass_idx<S2>(g, k)], then the Shoup companions at [L + i][g][k].
template <int LOGN>
__global__ void k_perm_s(const uint32_t* __restrict__ s_ntt, Rns R, uint32_t* __restrict__ s_enc) {
    using G = EncGeo<LOGN>;
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
    if (idx >= G::N) return;
    const uint32_t g = idx / 16, k = idx % 16;
    const uint32_t v = s_ntt[(size_t)i * G::N + pass_idx<G::S2>(g, k)];
    s_enc[(size_t)i * G::N + idx] = v;
    s_enc[(size_t)(R.L + i) * G::N + idx] = (uint32_t)(((uint64_t)v << 32) / R.p[i]);
}

// ---------------------------------------------------------------- launchers
bool encrypt_planes_ok(const nimbus_ctx* c) {
    const char* v = getenv("NIMBUS_ENC_TWOPASS");     // diagnostic: the two-pass path for A/B runs
    return (c->rns.N == 4096 || c->rns.N == 8192) && !(v && atoi(v) == 1);
}

cudaError_t launch_perm_s(nimbus_ctx* c, const uint32_t* d_s_ntt, uint32_t* d_s_enc, cudaStream_t st) {
    const dim3 g(c->rns.N / 256, c->rns.L);
    if (c->rns.N == 8192) k_perm_s<13><<<g, 256, 0, st>>>(d_s_ntt, c->rns, d_s_enc);
    else k_perm_s<12><<<g, 256, 0, st>>>(d_s_ntt, c->rns, d_s_enc);
    c->launches++;
    return cudaGetLastError();
}

template <int LOGN, typename TW>
static cudaError_t launch_enc_t(nimbus_ctx* c, const uint32_t* d_s_enc, const TW* d_W, uint32_t m, uint32_t n,
                                uint64_t seed, uint32_t KB, uint32_t bn, uint8_t* d_Et, cudaStream_t st) {
    using G = EncGeo<LOGN>;
    auto kern = k_encrypt_planes<LOGN, TW>;
    const size_t smem = (size_t)3 * G::N * 4;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && kEncRows > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(KB * kBK, c->rns.L);
    cfg.blockDim = dim3(G::T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kEncRows;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, c->rns, (const uint32_t*)c->d_tw, d_s_enc, d_W, m, n, seed, KB, bn, d_Et);
    c->launches++;
    return e;
}

cudaError_t launch_encrypt_planes(nimbus_ctx* c, const uint32_t* d_s_enc, const void* d_W, uint32_t m, uint32_t n,
                                  uint64_t seed, uint32_t KB, uint32_t bn, uint8_t* d_Et, cudaStream_t st) {
    // columns past 2 L N in the last tiles are zero padding the kernel does not write
    const uint32_t ncol = 2 * c->rns.L * c->rns.N, t0 = ncol / bn, tiles = col_tiles(c, bn);
    if (tiles > t0) {
        const size_t tile_bytes = (size_t)KB * kSW * bn * kBK;
        cudaError_t e = cudaMemsetAsync(d_Et + (size_t)t0 * tile_bytes, 0, (size_t)(tiles - t0) * tile_bytes, st);
        if (e != cudaSuccess) return e;
    }
    const bool w64 = elem_bytes(c->rns.ell) == 8;
    if (c->rns.N == 8192)
        return w64 ? launch_enc_t<13>(c, d_s_enc, static_cast<const uint64_t*>(d_W), m, n, seed, KB, bn, d_Et, st)
                   : launch_enc_t<13>(c, d_s_enc, static_cast<const uint32_t*>(d_W), m, n, seed, KB, bn, d_Et, st);
    return w64 ? launch_enc_t<12>(c, d_s_enc, static_cast<const uint64_t*>(d_W), m, n, seed, KB, bn, d_Et, st)
               : launch_enc_t<12>(c, d_s_enc, static_cast<const uint32_t*>(d_W), m, n, seed, KB, bn, d_Et, st);
}

}  // namespace nimbus
