// ntt.cu -- negacyclic NTT over Z_p[X]/(X^N+1) (§3.1; used only
// for KeyGen/Encrypt at setup and for the verification decrypt
// "the NTT is only applied when the server decrypts"), plus the KeyGen (K1),
// fused Encrypt-rows (K3) and Decrypt (K8) kernels.
//
// One CTA per (polynomial, limb); the N residues are staged in shared memory
// and transformed in place: Cooley-Tukey forward (natural -> bit-reversed) and
// Gentleman-Sande inverse (bit-reversed -> natural) with the negacyclic twist
// psi^i folded into the twiddles, Shoup modular multiplication.
#include "ntt_dev.cuh"

namespace nimbus {

// Cooley-Tukey forward, natural -> bit-reversed order
__device__ void ntt_fwd_smem(uint32_t* a, const uint32_t* tw, const uint32_t* tw_sh, uint32_t N,
                             uint32_t logN, uint32_t p) {
    uint32_t m = 1, lt = logN - 1;            // stage (m, t = 2^lt): pairs (j, j + t) in blocks of 2t
    for (; lt >= 1; m <<= 2, lt -= 2) {       // stages (m, t) and (2m, t/2)
        const uint32_t t = 1u << lt, h = t >> 1;
        for (uint32_t idx = threadIdx.x; idx < N / 4; idx += blockDim.x) {
            const uint32_t i = idx >> (lt - 1), j = idx & (h - 1);
            const uint32_t base = (i << (lt + 1)) + j;
            uint32_t x0 = a[base], x1 = a[base + h], x2 = a[base + t], x3 = a[base + t + h];
            const uint32_t S = tw[m + i], Ssh = tw_sh[m + i];
            ct_bfly(x0, x2, S, Ssh, p);
            ct_bfly(x1, x3, S, Ssh, p);
            const uint32_t k0 = 2 * m + 2 * i;
            ct_bfly(x0, x1, tw[k0], tw_sh[k0], p);
            ct_bfly(x2, x3, tw[k0 + 1], tw_sh[k0 + 1], p);
            a[base] = x0; a[base + h] = x1; a[base + t] = x2; a[base + t + h] = x3;
        }
        __syncthreads();
        if (lt == 1) { m <<= 2; lt = 0; break; }
    }
    if (m < N) {                               // odd log N: last radix-2 stage, t = 1
        for (uint32_t idx = threadIdx.x; idx < N / 2; idx += blockDim.x) {
            const uint32_t j1 = idx << 1;
            uint32_t x = a[j1], y = a[j1 + 1];
            ct_bfly(x, y, tw[m + idx], tw_sh[m + idx], p);
            a[j1] = x; a[j1 + 1] = y;
        }
        __syncthreads();
    }
}

// Gentleman-Sande inverse, bit-reversed -> natural order, times N^-1 if `scale`
__device__ void ntt_inv_smem(uint32_t* a, const uint32_t* itw, const uint32_t* itw_sh, uint32_t N,
                             uint32_t logN, uint32_t p, uint32_t ninv, uint32_t ninv_sh, bool scale = true) {
    uint32_t lt = 0, hh = N >> 1;             // stage (t = 2^lt, h = N / 2^(lt+1)): twiddle itw[h + i]
    if (logN & 1) {                            // odd log N: first radix-2 stage, t = 1
        for (uint32_t idx = threadIdx.x; idx < N / 2; idx += blockDim.x) {
            const uint32_t j1 = idx << 1;
            uint32_t x = a[j1], y = a[j1 + 1];
            gs_bfly(x, y, itw[hh + idx], itw_sh[hh + idx], p);
            a[j1] = x; a[j1 + 1] = y;
        }
        __syncthreads();
        lt = 1; hh >>= 1;
    }
    for (; (1u << lt) < N; lt += 2, hh >>= 2) {     // stages (t, h) and (2t, h/2)
        const uint32_t t = 1u << lt;
        for (uint32_t idx = threadIdx.x; idx < N / 4; idx += blockDim.x) {
            const uint32_t i = idx >> lt, j = idx & (t - 1);     // block of 4t
            const uint32_t base = (i << (lt + 2)) + j;
            uint32_t y0 = a[base], y1 = a[base + t], y2 = a[base + 2 * t], y3 = a[base + 3 * t];
            const uint32_t k0 = hh + 2 * i;
            gs_bfly(y0, y1, itw[k0], itw_sh[k0], p);
            gs_bfly(y2, y3, itw[k0 + 1], itw_sh[k0 + 1], p);
            const uint32_t k1 = (hh >> 1) + i;
            gs_bfly(y0, y2, itw[k1], itw_sh[k1], p);
            gs_bfly(y1, y3, itw[k1], itw_sh[k1], p);
            if (scale && (4u << lt) == N) {       // last pass: scale by N^-1 here
                y0 = mulmod_shoup(y0, ninv, ninv_sh, p);
                y1 = mulmod_shoup(y1, ninv, ninv_sh, p);
                y2 = mulmod_shoup(y2, ninv, ninv_sh, p);
                y3 = mulmod_shoup(y3, ninv, ninv_sh, p);
            }
            a[base] = y0; a[base + t] = y1; a[base + 2 * t] = y2; a[base + 3 * t] = y3;
        }
        __syncthreads();
    }
}

struct TwLimb {
    const uint32_t *fw, *fw_sh, *iv, *iv_sh;
};
__device__ __forceinline__ TwLimb tw_limb(const uint32_t* d_tw, uint32_t N, uint32_t i) {
    const uint32_t* b = d_tw + (size_t)i * 4 * N;
    return {b, b + N, b + 2 * N, b + 3 * N};
}
// Stage a limb's twiddle tables (forward pair, and the inverse pair if `inv`) in
// shared memory at `dst`: every butterfly stage then reads them without a global
// round trip (a transform is 2 log N dependent stages).  Returns the smem view.
__device__ __forceinline__ TwLimb tw_stage(const uint32_t* d_tw, uint32_t N, uint32_t i, uint32_t* dst, bool inv) {
    const uint4* src = reinterpret_cast<const uint4*>(d_tw + (size_t)i * 4 * N);
    uint4* d = reinterpret_cast<uint4*>(dst);
    const uint32_t n4 = (inv ? 4 * N : 2 * N) / 4;
    for (uint32_t j = threadIdx.x; j < n4; j += blockDim.x) d[j] = __ldg(src + j);
    return {dst, dst + N, dst + 2 * N, dst + 3 * N};
}

// ---------------------------------------------------------------- KeyGen (A1)
// s[j] = floor(word(seed,1,j) * 3 / 2^64) - 1; s_ntt[i] = NTT_{p_i}(s mod p_i)
__global__ void k_keygen(Rns R, const uint32_t* d_tw, uint64_t seed, int8_t* s, uint32_t* s_ntt) {
    extern __shared__ uint32_t sa[];
    const uint32_t N = R.N, i = blockIdx.x, p = R.p[i];
    const uint64_t key = prg_key(seed, 1);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) {
        int32_t v = samp_ternary(prg_word(key, j));
        if (i == 0) s[j] = (int8_t)v;
        sa[j] = v < 0 ? p - 1 : (uint32_t)v;
    }
    TwLimb tw = tw_stage(d_tw, N, i, sa + N, false);
    __syncthreads();
    ntt_fwd_smem(sa, tw.fw, tw.fw_sh, N, R.logN, p);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) s_ntt[(size_t)i * N + j] = sa[j];
}

// ---------------------------------------------------------------- Encrypt (A2)
// Alg. 1 step 1 for row beta = blockIdx.x, limb i = blockIdx.y:
//   a = uniform mod p_i (domain 2, index (beta L + i) N + j)
//   b = a*s + Emb_q(w_hat) + e mod p_i, e = CBD(21) (domain 3, index beta N + j),
//   w_hat[j] = W[beta][j] for j < n else 0 (Eq. 2).
// Writes the canonical layout encW[beta][comp][limb][j].
template <typename T>
__global__ void k_encrypt(Rns R, const uint32_t* d_tw, const uint32_t* s_ntt, const T* W,
                          uint32_t n, uint64_t seed, uint32_t* encW) {
    extern __shared__ uint32_t sa[];
    const uint32_t N = R.N, L = R.L, beta = blockIdx.x, i = blockIdx.y, p = R.p[i];
    const uint64_t mu = R.mu[i];
    const uint64_t ka = prg_key(seed, 2), ke = prg_key(seed, 3);
    uint32_t* bo = encW + (((size_t)beta * 2 + 0) * L + i) * N;
    uint32_t* ao = encW + (((size_t)beta * 2 + 1) * L + i) * N;
    // PRG counters stepped per thread: word(key, idx) = mix64(key + golden (idx + 1))
    constexpr uint64_t G = 0x9E3779B97F4A7C15ULL;
    const uint64_t dz = G * blockDim.x;
    uint64_t za = ka + G * (((uint64_t)beta * L + i) * N + threadIdx.x + 1);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x, za += dz) {
        uint32_t a = samp_uniform_mod(mix64(za), p);
        sa[j] = a;
        ao[j] = a;
    }
    // twiddles straight from global memory (L1/L2 resident): setup runs m x L CTAs,
    // and occupancy hides their latency better than staging them in shared memory
    TwLimb tw = tw_limb(d_tw, N, i);
    __syncthreads();
    ntt_fwd_smem(sa, tw.fw, tw.fw_sh, N, R.logN, p);
    const uint32_t* sn = s_ntt + (size_t)i * N;
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) sa[j] = mulmod(sa[j], sn[j], p, mu);
    __syncthreads();
    ntt_inv_smem(sa, tw.iv, tw.iv_sh, N, R.logN, p, R.ninv[i], R.ninv_sh[i]);
    uint64_t ze = ke + G * ((uint64_t)beta * N + threadIdx.x + 1);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x, ze += dz) {
        const uint64_t w = j < n ? (uint64_t)W[(size_t)beta * n + j] : 0u;
        int32_t e = samp_cbd21(mix64(ze));
        // Emb_q(w) mod p: 32-bit Shoup forms up to ell = 32, the 64-bit one beyond
        uint32_t em = R.ell > 32 ? emb_mod(w, R.q_mod_t, R.ell, p, mu, R.t_inv[i])
                      : R.ell <= 16 ? emb_fast16((uint32_t)w, (uint32_t)R.q_mod_t, R.ell, p, R.t_inv[i], R.t_inv_sh[i])
                                    : emb_fast((uint32_t)w, (uint32_t)R.q_mod_t, R.ell, p, R.t_inv[i], R.t_inv_sh[i]);
        uint32_t er = e < 0 ? p - (uint32_t)(-e) : (uint32_t)e;
        bo[j] = addmod(addmod(sa[j], em, p), er, p);
    }
}

// ---------------------------------------------------------------- public key (reading 25)
// PAPER.md:602 KeyGen "(sk, pk)": limb i = blockIdx.x,
//   a = uniform mod p_i (domain 7, index i N + j), e = CBD(21) (domain 8, index j),
//   b = a*s + e mod p_i.  Writes pk[comp b=0, a=1][limb][j] (coefficients).
__global__ void k_keygen_pk(Rns R, const uint32_t* d_tw, const uint32_t* s_ntt, uint64_t seed, uint32_t* pk) {
    extern __shared__ uint32_t sa[];
    const uint32_t N = R.N, L = R.L, i = blockIdx.x, p = R.p[i];
    const uint64_t ka = prg_key(seed, 7), ke = prg_key(seed, 8);
    uint32_t* bo = pk + (size_t)i * N;
    uint32_t* ao = pk + ((size_t)L + i) * N;
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) {
        const uint32_t a = samp_uniform_mod(prg_word(ka, (uint64_t)i * N + j), p);
        sa[j] = a;
        ao[j] = a;
    }
    TwLimb tw = tw_limb(d_tw, N, i);
    __syncthreads();
    ntt_fwd_smem(sa, tw.fw, tw.fw_sh, N, R.logN, p);
    const uint32_t* sn = s_ntt + (size_t)i * N;
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) sa[j] = mulmod(sa[j], sn[j], p, R.mu[i]);
    __syncthreads();
    ntt_inv_smem(sa, tw.iv, tw.iv_sh, N, R.logN, p, R.ninv[i], R.ninv_sh[i]);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) {
        const int32_t e = samp_cbd21(prg_word(ke, j));
        bo[j] = addmod(sa[j], e < 0 ? p - (uint32_t)(-e) : (uint32_t)e, p);
    }
}

// forward NTT of polynomial blockIdx.x, limb blockIdx.y of a [count][L][N] array
__global__ void k_ntt_rows(Rns R, const uint32_t* d_tw, const uint32_t* in, uint32_t* out) {
    extern __shared__ uint32_t sa[];
    const uint32_t N = R.N, i = blockIdx.y, p = R.p[i];
    const size_t off = ((size_t)blockIdx.x * R.L + i) * N;
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) sa[j] = in[off + j];
    TwLimb tw = tw_limb(d_tw, N, i);
    __syncthreads();
    ntt_fwd_smem(sa, tw.fw, tw.fw_sh, N, R.logN, p);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) out[off + j] = sa[j];
}

// signed 64-bit value mod p
__device__ __forceinline__ uint32_t smod64(int64_t e, uint32_t p) {
    const uint64_t mag = e < 0 ? (uint64_t)(-(e + 1)) + 1 : (uint64_t)e;
    const uint32_t r = (uint32_t)(mag % p);
    return (e < 0 && r) ? p - r : r;
}

// ---------------------------------------------------------------- circuit privacy (reading 26)
// the client's output must not reveal X_c to the key owner.  One
// public-key encryption of zero per packed ciphertext g = blockIdx.x, limb i = blockIdx.y:
//   v ternary (domain 9, index g N + j), e1, e2 CBD(21) (domains 10, 11, index g N + j),
//   f flooding noise (w >> (63 - F)) - 2^F (domain 12; none when F = 0),
//   z_b = v b_pk + e1 + f,  z_a = v a_pk + e2  mod p_i   ->  z[g][comp][limb][j].
// Offline (input-independent) work: the online pack only adds z before its ModDown.
__global__ void k_rerand(Rns R, const uint32_t* d_tw, const uint32_t* pk_ntt, uint64_t seed, uint32_t F,
                         uint32_t* z) {
    extern __shared__ uint32_t sm[];
    const uint32_t N = R.N, L = R.L, g = blockIdx.x, i = blockIdx.y, p = R.p[i];
    uint32_t *sv = sm, *sp = sm + N;
    const uint64_t kv = prg_key(seed, 9), k1 = prg_key(seed, 10), k2 = prg_key(seed, 11), kf = prg_key(seed, 12),
                   kf2 = prg_key(seed, 13);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) {
        const int32_t v = samp_ternary(prg_word(kv, (uint64_t)g * N + j));
        sv[j] = v < 0 ? p - 1 : (uint32_t)v;
    }
    TwLimb tw = tw_limb(d_tw, N, i);
    __syncthreads();
    ntt_fwd_smem(sv, tw.fw, tw.fw_sh, N, R.logN, p);
    for (uint32_t comp = 0; comp < 2; comp++) {
        const uint32_t* pn = pk_ntt + ((size_t)comp * L + i) * N;
        for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) sp[j] = mulmod(sv[j], pn[j], p, R.mu[i]);
        __syncthreads();
        ntt_inv_smem(sp, tw.iv, tw.iv_sh, N, R.logN, p, R.ninv[i], R.ninv_sh[i]);
        uint32_t* zo = z + (((size_t)g * 2 + comp) * L + i) * N;
        for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) {
            const uint64_t idx = (uint64_t)g * N + j;
            int64_t e;
            uint32_t fm = 0;                          // flooding noise mod p (reading 26)
            if (comp == 0) {
                e = samp_cbd21(prg_word(k1, idx));
                if (F && F <= 62) {
                    e += (int64_t)(prg_word(kf, idx) >> (63 - F)) - ((int64_t)1 << F);
                } else if (F > 62) {
                    // f = (V >> (127 - F)) - 2^F, V = w1 2^64 + w0 (domains 13, 12): f mod p from 128 bits
                    const unsigned __int128 V = ((unsigned __int128)prg_word(kf2, idx) << 64) | prg_word(kf, idx);
                    const unsigned __int128 top = V >> (127 - F);
                    const uint32_t tm = (uint32_t)(top % p), pw = (uint32_t)((((unsigned __int128)1) << F) % p);
                    fm = submod(tm, pw, p);
                }
            } else {
                e = samp_cbd21(prg_word(k2, idx));
            }
            zo[j] = addmod(addmod(sp[j], smod64(e, p), p), fm, p);
        }
        __syncthreads();   // sp is reused by the next component
    }
}

// ---------------------------------------------------------------- test helper
__global__ void k_negacyclic_mul(Rns R, const uint32_t* d_tw, const uint32_t* A, const uint32_t* B,
                                 uint32_t* Cout) {
    extern __shared__ uint32_t sm[];
    const uint32_t N = R.N, i = blockIdx.y, p = R.p[i];
    uint32_t *sa = sm, *sb = sm + N;
    const size_t off = ((size_t)blockIdx.x * R.L + i) * N;
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) { sa[j] = A[off + j]; sb[j] = B[off + j]; }
    TwLimb tw = tw_stage(d_tw, N, i, sm + 2 * N, true);
    __syncthreads();
    ntt_fwd_smem(sa, tw.fw, tw.fw_sh, N, R.logN, p);
    ntt_fwd_smem(sb, tw.fw, tw.fw_sh, N, R.logN, p);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) sa[j] = mulmod(sa[j], sb[j], p, R.mu[i]);
    __syncthreads();
    ntt_inv_smem(sa, tw.iv, tw.iv_sh, N, R.logN, p, R.ninv[i], R.ninv_sh[i]);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) Cout[off + j] = sa[j];
}

// ---------------------------------------------------------------- Decrypt (A7)
// Per packed ciphertext tg and limb i < L_out: u_i = b_i - a_i * s mod p_i.
__global__ void k_decrypt_phase(Rns R, const uint32_t* d_tw, const uint32_t* s_ntt, const uint32_t* cts,
                                uint32_t* U) {
    extern __shared__ uint32_t sa[];
    const uint32_t N = R.N, Lo = R.L_out, tg = blockIdx.x, i = blockIdx.y, p = R.p[i];
    const uint32_t* b = cts + (((size_t)tg * 2 + 0) * Lo + i) * N;
    const uint32_t* a = cts + (((size_t)tg * 2 + 1) * Lo + i) * N;
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) sa[j] = a[j];
    TwLimb tw = tw_stage(d_tw, N, i, sa + N, true);
    __syncthreads();
    ntt_fwd_smem(sa, tw.fw, tw.fw_sh, N, R.logN, p);
    const uint32_t* sn = s_ntt + (size_t)i * N;
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) sa[j] = mulmod(sa[j], sn[j], p, R.mu[i]);
    __syncthreads();
    ntt_inv_smem(sa, tw.iv, tw.iv_sh, N, R.logN, p, R.ninv[i], R.ninv_sh[i]);
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) U[((size_t)tg * Lo + i) * N + j] = submod(b[j], sa[j], p);
}

// Same, one polynomial per 4-CTA cluster: CTA r holds coefficients [r Q, (r+1) Q),
// Q = N/4, in shared memory.  The two forward stages and the two inverse stages
// whose butterflies span the quarters run as one radix-4 pass over distributed
// shared memory (each CTA takes a quarter of the Q four-element groups); every
// other stage is CTA-local.  4x the SMs per polynomial: a few dozen packed
// ciphertexts (C2: 26) no longer leave most of the GPU idle.
constexpr uint32_t kDecCl = 4;

// With one output limb (L_out = 1, ell <= 32) the rounding and unpacking of
// k_decrypt_round are done here too (Z, M non-null; U unused): q' = p_0, so
// m = floor((2 t u + p_0) / (2 p_0)) fits 64-bit arithmetic.
__global__ void __launch_bounds__(256) k_decrypt_cl(Rns R, const uint32_t* d_tw, const uint32_t* s_ntt,
                                                   const uint32_t* cts, uint32_t* U, uint32_t nct, uint32_t kq,
                                                   uint32_t n, uint32_t* Z, uint32_t* M) {
    extern __shared__ uint32_t sa[];
    const uint32_t N = R.N, Q = N / kDecCl, logQ = R.logN - 2, Lo = R.L_out;
    const uint32_t r = cluster_ctarank(), tg = blockIdx.x / kDecCl, i = blockIdx.y, p = R.p[i];
    const uint32_t* b = cts + (((size_t)tg * 2 + 0) * Lo + i) * N + r * Q;
    const uint32_t* a = cts + (((size_t)tg * 2 + 1) * Lo + i) * N + r * Q;
    for (uint32_t j = threadIdx.x; j < Q; j += blockDim.x) sa[j] = a[j];
    const TwLimb tw = tw_limb(d_tw, N, i);
    // this CTA's local-stage twiddles, re-indexed as a length-Q table: its stage-m
    // block i is block r m + i of the global stage 4m, whose twiddle is entry
    // 4m + r m + i; stored at m + i, the local stages run as a plain length-Q NTT
    uint32_t* st = sa + Q;                        // [fw | fw_sh | iv | iv_sh], Q words each
    for (uint32_t e = threadIdx.x; e < Q; e += blockDim.x) {
        if (e == 0) continue;
        const uint32_t m = 1u << (31 - __clz(e)), g = m * (kDecCl + r) + (e - m);
        st[e] = tw.fw[g]; st[Q + e] = tw.fw_sh[g]; st[2 * Q + e] = tw.iv[g]; st[3 * Q + e] = tw.iv_sh[g];
    }
    uint32_t rem[kDecCl];
#pragma unroll
    for (uint32_t c = 0; c < kDecCl; c++) rem[c] = dsmem_addr(sa, c);
    cluster_sync();
    // forward stages (m = 1, t = N/2) and (m = 2, t = N/4): group j = {j, j+Q, j+2Q, j+3Q}
    {
        const uint32_t S1 = tw.fw[1], S1s = tw.fw_sh[1], S2 = tw.fw[2], S2s = tw.fw_sh[2];
        const uint32_t S3 = tw.fw[3], S3s = tw.fw_sh[3];
        for (uint32_t j = r * (Q / kDecCl) + threadIdx.x; j < (r + 1) * (Q / kDecCl); j += blockDim.x) {
            uint32_t x0 = ld_dsmem(rem[0] + 4 * j), x1 = ld_dsmem(rem[1] + 4 * j);
            uint32_t x2 = ld_dsmem(rem[2] + 4 * j), x3 = ld_dsmem(rem[3] + 4 * j);
            ct_bfly(x0, x2, S1, S1s, p);
            ct_bfly(x1, x3, S1, S1s, p);
            ct_bfly(x0, x1, S2, S2s, p);
            ct_bfly(x2, x3, S3, S3s, p);
            st_dsmem(rem[0] + 4 * j, x0); st_dsmem(rem[1] + 4 * j, x1);
            st_dsmem(rem[2] + 4 * j, x2); st_dsmem(rem[3] + 4 * j, x3);
        }
    }
    cluster_sync();
    ntt_fwd_smem(sa, st, st + Q, Q, logQ, p);
    const uint32_t* sn = s_ntt + (size_t)i * N + r * Q;
    for (uint32_t j = threadIdx.x; j < Q; j += blockDim.x) sa[j] = mulmod(sa[j], sn[j], p, R.mu[i]);
    __syncthreads();
    ntt_inv_smem(sa, st + 2 * Q, st + 3 * Q, Q, logQ, p, 0, 0, false);
    cluster_sync();
    // inverse stages (t = N/4, h = 2) and (t = N/2, h = 1), then N^-1
    {
        const uint32_t S1 = tw.iv[1], S1s = tw.iv_sh[1], S2 = tw.iv[2], S2s = tw.iv_sh[2];
        const uint32_t S3 = tw.iv[3], S3s = tw.iv_sh[3], ni = R.ninv[i], nis = R.ninv_sh[i];
        for (uint32_t j = r * (Q / kDecCl) + threadIdx.x; j < (r + 1) * (Q / kDecCl); j += blockDim.x) {
            uint32_t y0 = ld_dsmem(rem[0] + 4 * j), y1 = ld_dsmem(rem[1] + 4 * j);
            uint32_t y2 = ld_dsmem(rem[2] + 4 * j), y3 = ld_dsmem(rem[3] + 4 * j);
            gs_bfly(y0, y1, S2, S2s, p);
            gs_bfly(y2, y3, S3, S3s, p);
            gs_bfly(y0, y2, S1, S1s, p);
            gs_bfly(y1, y3, S1, S1s, p);
            st_dsmem(rem[0] + 4 * j, mulmod_shoup(y0, ni, nis, p));
            st_dsmem(rem[1] + 4 * j, mulmod_shoup(y1, ni, nis, p));
            st_dsmem(rem[2] + 4 * j, mulmod_shoup(y2, ni, nis, p));
            st_dsmem(rem[3] + 4 * j, mulmod_shoup(y3, ni, nis, p));
        }
    }
    cluster_sync();
    if (Z) {                                  // L_out = 1: round and unpack here
        const uint32_t ell = R.ell, Rr = N / n, theta = tg % nct, query = tg / nct;
        const uint32_t rows = min(Rr, kq - theta * Rr);
        const uint64_t tmask = (1ULL << ell) - 1;
        for (uint32_t j = threadIdx.x; j < Q; j += blockDim.x) {
            const uint32_t J = r * Q + j, u = submod(b[j], sa[j], p);
            const uint32_t m = (uint32_t)(((((uint64_t)u << (ell + 1)) + p) / (2ULL * p)) & tmask);
            if (M) M[(size_t)tg * N + J] = m;
            if (J < rows * n) Z[((size_t)query * kq + theta * Rr) * n + J] = m;
        }
        return;
    }
    uint32_t* u = U + ((size_t)tg * Lo + i) * N + r * Q;
    for (uint32_t j = threadIdx.x; j < Q; j += blockDim.x) u[j] = submod(b[j], sa[j], p);
}

// CRT (Garner) of u_0..u_{Lo-1} and m = floor((2 t u + q') / (2 q')) mod t
// (SURVEY.md §8(c) #5); unpack Z[alpha][j] = m_theta[(alpha mod R) n + j].
// The division is exact long division in 32-bit steps on 128-bit words
// (u < q' < 2^95, t <= 2^64: 2 t u alone can exceed 128 bits).  T = uint32_t,
// or uint64_t for ell > 32.
template <typename T>
__global__ void k_decrypt_round(Rns R, const uint32_t* U, uint32_t nct, uint32_t kq, uint32_t n,
                                T* Z, T* M, u128 qout, uint32_t garner0, uint32_t garner1) {
    const uint32_t N = R.N, Lo = R.L_out, tg = blockIdx.y;
    const uint32_t J = blockIdx.x * blockDim.x + threadIdx.x;
    if (J >= N) return;
    // Garner: u = v0 + p0 (v1 + p1 v2), v_i in [0, p_i)
    uint32_t u0 = U[((size_t)tg * Lo + 0) * N + J];
    u128 u = u0;
    if (Lo >= 2) {
        uint32_t p1 = R.p[1];
        uint32_t u1 = U[((size_t)tg * Lo + 1) * N + J];
        // v1 = (u1 - u0) * p0^-1 mod p1
        uint32_t v1 = mulmod(submod(u1, u0 % p1, p1), garner0, p1, R.mu[1]);
        u += (u128)R.p[0] * v1;
        if (Lo >= 3) {
            uint32_t p2 = R.p[2];
            uint32_t u2 = U[((size_t)tg * Lo + 2) * N + J];
            // v2 = (u2 - (u0 + p0 v1)) * (p0 p1)^-1 mod p2
            uint64_t x = (uint64_t)u0 + (uint64_t)R.p[0] * v1;  // < 2^62
            uint32_t xm = mod64(x, p2, R.mu[2]);
            uint32_t v2 = mulmod(submod(u2, xm, p2), garner1, p2, R.mu[2]);
            u += (u128)R.p[0] * R.p[1] * v2;
        }
    }
    const uint32_t ell = R.ell;
    // u 2^(ell+1) = Q (2 q') + r by shifting the remainder 32 bits at a time (r < 2q' < 2^96)
    const u128 den = qout << 1;
    u128 Q = 0, r = u;
    for (uint32_t S = ell + 1; S > 0;) {
        const uint32_t sh = S < 32 ? S : 32;
        r <<= sh;
        Q = (Q << sh) + r / den;
        r %= den;
        S -= sh;
    }
    Q += (r + qout) / den;                                  // + q', then floor
    const uint64_t tmask = ell >= 64 ? ~0ULL : ((1ULL << ell) - 1);
    const T m = (T)((uint64_t)Q & tmask);
    if (M) M[(size_t)tg * N + J] = m;
    const uint32_t Rr = N / n, theta = tg % nct, query = tg / nct;
    const uint32_t rows = min(Rr, kq - theta * Rr);
    if (J < rows * n) Z[((size_t)query * kq + theta * Rr) * n + J] = m;
}

__global__ void k_prg_words(uint64_t seed, uint32_t dom, uint64_t start, uint64_t count, uint64_t* out) {
    const uint64_t key = prg_key(seed, dom);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = prg_word(key, start + i);
}

// ---------------------------------------------------------------- launchers
static uint32_t ntt_threads(uint32_t N) { return N >= 1024 ? 512 : N / 2; }

// dynamic shared memory of the NTT kernels: `words` 32-bit words (data + staged twiddles)
template <typename K>
static cudaError_t ntt_smem(K kernel, size_t words) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(words * 4));
}

cudaError_t launch_keygen(nimbus_ctx* c, uint64_t seed, int8_t* d_s, uint32_t* d_s_ntt, cudaStream_t st) {
    const uint32_t N = c->rns.N;
    cudaError_t e = ntt_smem(k_keygen, 3 * N);
    if (e != cudaSuccess) return e;
    k_keygen<<<c->rns.L, ntt_threads(N), 3 * N * 4, st>>>(c->rns, c->d_tw, seed, d_s, d_s_ntt);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_encrypt(nimbus_ctx* c, const uint32_t* d_s_ntt, const void* d_W, uint32_t m,
                           uint32_t n, uint64_t seed, uint32_t* d_encW, cudaStream_t st) {
    const uint32_t N = c->rns.N;
    if (elem_bytes(c->rns.ell) == 8)
        k_encrypt<uint64_t><<<dim3(m, c->rns.L), ntt_threads(N), N * 4, st>>>(
            c->rns, c->d_tw, d_s_ntt, static_cast<const uint64_t*>(d_W), n, seed, d_encW);
    else
        k_encrypt<uint32_t><<<dim3(m, c->rns.L), ntt_threads(N), N * 4, st>>>(
            c->rns, c->d_tw, d_s_ntt, static_cast<const uint32_t*>(d_W), n, seed, d_encW);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_keygen_pk(nimbus_ctx* c, const uint32_t* d_s_ntt, uint64_t seed, uint32_t* d_pk, cudaStream_t st) {
    const uint32_t N = c->rns.N;
    cudaError_t e = ntt_smem(k_keygen_pk, N);
    if (e != cudaSuccess) return e;
    k_keygen_pk<<<c->rns.L, ntt_threads(N), N * 4, st>>>(c->rns, c->d_tw, d_s_ntt, seed, d_pk);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_ntt_rows(nimbus_ctx* c, const uint32_t* in, uint32_t count, uint32_t* out, cudaStream_t st) {
    const uint32_t N = c->rns.N;
    cudaError_t e = ntt_smem(k_ntt_rows, N);
    if (e != cudaSuccess) return e;
    k_ntt_rows<<<dim3(count, c->rns.L), ntt_threads(N), N * 4, st>>>(c->rns, c->d_tw, in, out);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_rerand(nimbus_ctx* c, const uint32_t* d_pk_ntt, uint64_t seed, uint32_t n_cts, uint32_t F,
                          uint32_t* d_zero, cudaStream_t st) {
    const uint32_t N = c->rns.N;
    cudaError_t e = ntt_smem(k_rerand, 2 * N);
    if (e != cudaSuccess) return e;
    k_rerand<<<dim3(n_cts, c->rns.L), ntt_threads(N), 2 * N * 4, st>>>(c->rns, c->d_tw, d_pk_ntt, seed, F, d_zero);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_negacyclic_mul(nimbus_ctx* c, const uint32_t* a, const uint32_t* b, uint32_t count,
                                  uint32_t* out, cudaStream_t st) {
    const uint32_t N = c->rns.N;
    const size_t smem = (size_t)N * 6 * 4;
    cudaError_t e = ntt_smem(k_negacyclic_mul, 6 * N);
    if (e != cudaSuccess) return e;
    k_negacyclic_mul<<<dim3(count, c->rns.L), ntt_threads(N), smem, st>>>(c->rns, c->d_tw, a, b, out);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_decrypt(nimbus_ctx* c, const uint32_t* d_s_ntt, const uint32_t* cts, uint32_t nct_total,
                           uint32_t nct, uint32_t kq, uint32_t n, uint32_t* d_u_tmp, void* d_Z,
                           void* d_M, cudaStream_t st) {
    const uint32_t N = c->rns.N;
    {
        // one 4-CTA cluster per (ciphertext, limb), a quarter of the coefficients each
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nct_total * kDecCl, c->rns.L_out);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = (size_t)N / kDecCl * 5 * 4;     // quarter + its 4 twiddle tables
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kDecCl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        // L_out = 1 (ell <= 32): round and unpack inside the cluster kernel
        const bool fused = c->rns.L_out == 1 && elem_bytes(c->rns.ell) == 4;
        cudaError_t e0 = cudaLaunchKernelEx(&cfg, k_decrypt_cl, c->rns, (const uint32_t*)c->d_tw, d_s_ntt, cts,
                                            d_u_tmp, nct, kq, n, fused ? static_cast<uint32_t*>(d_Z) : nullptr,
                                            fused ? static_cast<uint32_t*>(d_M) : nullptr);
        if (e0 != cudaSuccess) return e0;
        c->launches++;
        if (fused) return cudaGetLastError();
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // Garner constants
    const nimbus::Rns& R = c->rns;
    auto inv = [](uint64_t a, uint64_t p) {
        uint64_t r = 1, e2 = p - 2; a %= p;
        while (e2) { if (e2 & 1) r = (uint64_t)((u128)r * a % p); a = (uint64_t)((u128)a * a % p); e2 >>= 1; }
        return (uint32_t)r;
    };
    uint32_t g0 = R.L_out >= 2 ? inv(R.p[0], R.p[1]) : 0;
    uint32_t g1 = R.L_out >= 3 ? inv((uint64_t)R.p[0] * R.p[1] % R.p[2], R.p[2]) : 0;
    const dim3 gr((N + 255) / 256, nct_total);
    if (elem_bytes(c->rns.ell) == 8)
        k_decrypt_round<uint64_t><<<gr, 256, 0, st>>>(c->rns, d_u_tmp, nct, kq, n, static_cast<uint64_t*>(d_Z),
                                                      static_cast<uint64_t*>(d_M), c->qout, g0, g1);
    else
        k_decrypt_round<uint32_t><<<gr, 256, 0, st>>>(c->rns, d_u_tmp, nct, kq, n, static_cast<uint32_t*>(d_Z),
                                                      static_cast<uint32_t*>(d_M), c->qout, g0, g1);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_prg_words(uint64_t seed, uint32_t dom, uint64_t start, uint64_t count, uint64_t* out,
                             cudaStream_t st) {
    k_prg_words<<<592, 256, 0, st>>>(seed, dom, start, count, out);
    return cudaGetLastError();
}

}  // namespace nimbus
