/*
 * nimbus_oracle.c -- plain, slow, obviously-correct CPU oracle for the Nimbus
 * client-side outer-product (COP) homomorphic matmul (arXiv 2411.15707).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code with the CUDA path (paper_2411_15707_b200/) and includes none
 * of its headers.  Every function cites the passage it follows:
 *   PAPER.md:<line>  = /root/reference/PAPER.md line (section / algorithm)
 *   SURVEY.md §8(c)  = the reading taken where the paper is silent (listed in
 *                      DESIGN.md "Readings of the paper").
 *
 * Arithmetic: exact integers.  Products of two residues < 2^31 fit in uint64;
 * anything that can exceed 2^64 (CRT values up to q ~ 2^93, q*w, t*u) uses
 * unsigned __int128.  No blocking, fusion or reordering beyond the definitions.
 *
 * Pinned by tests/test_oracle_pins.py (brute force, closed forms, round trips,
 * special cases).  Functions without an external pin say "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------- */
/* PRG contract (SURVEY.md App. B "PRG"; the paper draws its randomness from  */
/* an unspecified source, App. B.1 KeyGen/Encryption).       */
/* ------------------------------------------------------------------------- */
uint64_t orc_mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27; z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

uint64_t orc_word(uint64_t seed, uint32_t dom, uint64_t i) {
    uint64_t key = orc_mix64(seed ^ ((uint64_t)dom << 56));
    return orc_mix64(key + 0x9E3779B97F4A7C15ULL * (i + 1));
}

void orc_words(uint64_t seed, uint32_t dom, uint64_t start, uint64_t count, uint64_t* out) {
    for (uint64_t i = 0; i < count; i++) out[i] = orc_word(seed, dom, start + i);
}

/* samplers (SURVEY.md App. B "Samplers") */
static uint32_t uniform_mod(uint64_t w, uint32_t p) { return (uint32_t)(((u128)w * p) >> 64); }
static int32_t ternary(uint64_t w) { return (int32_t)(((u128)w * 3) >> 64) - 1; }
static int32_t cbd21(uint64_t w) {
    return __builtin_popcountll(w & 0x1FFFFFULL) - __builtin_popcountll((w >> 21) & 0x1FFFFFULL);
}
static uint32_t uniform_t(uint64_t w, uint32_t ell) { return (uint32_t)(w >> (64 - ell)); }

/* ------------------------------------------------------------------------- */
/* Integer helpers                                                            */
/* ------------------------------------------------------------------------- */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)((u128)a * b % p); }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p; a %= p;
    while (e) { if (e & 1) r = mulmod(r, a, p); a = mulmod(a, a, p); e >>= 1; }
    return r;
}
/* inverse mod prime p by Fermat */
static uint64_t invmod(uint64_t a, uint64_t p) { return powmod(a, p - 2, p); }
/* signed value v -> residue mod p in [0,p) */
static uint32_t smod(int64_t v, uint32_t p) { int64_t r = v % (int64_t)p; return (uint32_t)(r < 0 ? r + p : r); }

/* trial division; n < 2^32 */
int orc_is_prime(uint64_t n) {
    if (n < 2) return 0;
    for (uint64_t d = 2; d * d <= n; d++) if (n % d == 0) return 0;
    return 1;
}

/* q = product of the L largest primes p < 2^31 with
 * p = 1 mod 2N, listed in descending order (the paper never states q,
 * PAPER.md:600 App. B.1 "{N, q, t}").  Returns 0 on success. */
int orc_primes(uint32_t N, uint32_t L, uint32_t* out) {
    uint64_t step = 2ULL * N;
    uint64_t c = ((((1ULL << 31) - 1) - 1) / step) * step + 1; /* largest 1 mod 2N below 2^31 */
    uint32_t found = 0;
    while (found < L && c > step) {
        if (orc_is_prime(c)) out[found++] = (uint32_t)c;
        c -= step;
    }
    return found == L ? 0 : -1;
}

/* q = prod p_i as a 128-bit integer */
static u128 prod_q(const uint32_t* primes, uint32_t L) {
    u128 q = 1;
    for (uint32_t i = 0; i < L; i++) q *= primes[i];
    return q;
}

/* ------------------------------------------------------------------------- */
/* Negacyclic ring Z_p[X]/(X^N+1)  (§2.1 A_{N,2^l}; App. B.1    */
/* "Plaintext-ciphertext polynomial Multiplication")            */
/* ------------------------------------------------------------------------- */

/* Schoolbook definition: c[k] = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j. */
void orc_negacyclic_schoolbook(uint32_t N, uint32_t p, const uint32_t* a, const uint32_t* b, uint32_t* c) {
    for (uint32_t k = 0; k < N; k++) {
        uint64_t pos = 0, neg = 0;
        for (uint32_t i = 0; i < N; i++) {
            uint32_t j;
            if (i <= k) { j = k - i; pos = (pos + mulmod(a[i], b[j], p)) % p; }
            else        { j = k + N - i; neg = (neg + mulmod(a[i], b[j], p)) % p; }
        }
        c[k] = (uint32_t)((pos + p - neg) % p);
    }
}

/* psi: a primitive 2N-th root of unity mod p (psi^N = -1).  Any such root
 * gives the same product; the choice is not observable. */
static uint64_t find_psi(uint32_t N, uint32_t p) {
    for (uint64_t x = 2; x < p; x++) {
        uint64_t psi = powmod(x, (p - 1) / (2ULL * N), p);
        if (powmod(psi, N, p) == p - 1) return psi;
    }
    return 0;
}

static uint32_t bitrev(uint32_t x, uint32_t logn) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < logn; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* Textbook iterative radix-2 cyclic DFT over Z_p with root w of order n
 * (bit-reversal permutation, then log n butterfly passes). */
static void dft(uint64_t* v, uint32_t n, uint64_t w, uint64_t p) {
    uint32_t logn = 0; while ((1u << logn) < n) logn++;
    for (uint32_t i = 0; i < n; i++) {
        uint32_t j = bitrev(i, logn);
        if (j > i) { uint64_t t = v[i]; v[i] = v[j]; v[j] = t; }
    }
    for (uint32_t len = 2; len <= n; len <<= 1) {
        uint64_t wl = powmod(w, n / len, p);
        for (uint32_t s = 0; s < n; s += len) {
            uint64_t wk = 1;
            for (uint32_t j = 0; j < len / 2; j++) {
                uint64_t u = v[s + j], x = mulmod(v[s + j + len / 2], wk, p);
                v[s + j] = (u + x) % p;
                v[s + j + len / 2] = (u + p - x) % p;
                wk = mulmod(wk, wl, p);
            }
        }
    }
}

/* Negacyclic product via the twisted cyclic convolution:
 *   a'[j] = a[j] psi^j, b'[j] = b[j] psi^j, c' = IDFT(DFT(a') . DFT(b')) with
 *   omega = psi^2, c[j] = c'[j] psi^-j.  (NTT as used by the paper.) */
void orc_negacyclic_ntt(uint32_t N, uint32_t p, const uint32_t* a, const uint32_t* b, uint32_t* c) {
    uint64_t psi = find_psi(N, p), psi_inv = invmod(psi, p);
    uint64_t w = mulmod(psi, psi, p), w_inv = invmod(w, p), n_inv = invmod(N, p);
    uint64_t* A = (uint64_t*)malloc(sizeof(uint64_t) * N);
    uint64_t* B = (uint64_t*)malloc(sizeof(uint64_t) * N);
    uint64_t pw = 1;
    for (uint32_t j = 0; j < N; j++) { A[j] = mulmod(a[j], pw, p); B[j] = mulmod(b[j], pw, p); pw = mulmod(pw, psi, p); }
    dft(A, N, w, p); dft(B, N, w, p);
    for (uint32_t j = 0; j < N; j++) A[j] = mulmod(A[j], B[j], p);
    dft(A, N, w_inv, p);
    pw = 1;
    for (uint32_t j = 0; j < N; j++) { c[j] = (uint32_t)mulmod(mulmod(A[j], n_inv, p), pw, p); pw = mulmod(pw, psi_inv, p); }
    free(A); free(B);
}

/* ------------------------------------------------------------------------- */
/* RLWE KeyGen / Encrypt / Decrypt (App. B.1)               */
/* ------------------------------------------------------------------------- */

/* KeyGen: ternary secret s, uniform over {-1,0,1} (SURVEY.md §8(c) #7, #8:
 * symmetric key, the server encrypts its own weights). */
void orc_keygen(uint32_t N, uint64_t seed, int8_t* s) {
    for (uint32_t j = 0; j < N; j++) s[j] = (int8_t)ternary(orc_word(seed, 1, j));
}

/* Emb_q(w) = floor((q*w + t/2) / t)  (reduces to the
 * Delta*w of an exact q/t when t | q). */
static u128 emb(u128 q, uint64_t w, uint32_t ell) {
    /* floor((q w + t/2) / t) evaluated without forming q w (which exceeds
     * 128 bits for 4 limbs): q = a t + b  =>  a w + floor((b w + t/2) / t). */
    u128 t = (u128)1 << ell;
    u128 a = q >> ell, b = q & (t - 1);
    return a * w + (b * w + t / 2) / t;
}

/* Encrypt the row-wise encoded weight rows (Alg. 1 step 1, PAPER.md:663;
 * row-wise encoding Eq. 2: w_hat[j] = W[beta][j] for j < n,
 * 0 for n <= j < N).  For each beta and limb i:
 *   a_i = uniform mod p_i (domain 2), e = CBD(21) (domain 3, one integer poly),
 *   b_i = a_i * s + Emb_q(w_hat) + e  mod p_i.
 * Output canonical layout encW[beta][comp b=0,a=1][limb][j]. */
void orc_encrypt_rows(uint32_t N, uint32_t L, const uint32_t* primes, uint32_t ell, const int8_t* s,
                      const uint32_t* W, uint32_t m, uint32_t n, uint64_t seed, uint32_t* encW) {
    u128 q = prod_q(primes, L);
    #pragma omp parallel for schedule(dynamic)
    for (int64_t beta = 0; beta < (int64_t)m; beta++) {
        uint32_t* a = (uint32_t*)malloc(4ULL * N);
        uint32_t* sv = (uint32_t*)malloc(4ULL * N);
        uint32_t* as = (uint32_t*)malloc(4ULL * N);
        int32_t* e = (int32_t*)malloc(4ULL * N);
        for (uint32_t j = 0; j < N; j++) e[j] = cbd21(orc_word(seed, 3, (uint64_t)beta * N + j));
        for (uint32_t i = 0; i < L; i++) {
            uint32_t p = primes[i];
            for (uint32_t j = 0; j < N; j++) {
                a[j] = uniform_mod(orc_word(seed, 2, ((uint64_t)beta * L + i) * N + j), p);
                sv[j] = smod(s[j], p);
            }
            orc_negacyclic_ntt(N, p, a, sv, as);
            uint32_t* bo = encW + (((uint64_t)beta * 2 + 0) * L + i) * N;
            uint32_t* ao = encW + (((uint64_t)beta * 2 + 1) * L + i) * N;
            for (uint32_t j = 0; j < N; j++) {
                uint64_t w = (j < n) ? W[(uint64_t)beta * n + j] : 0;
                uint64_t embv = (uint64_t)(emb(q, w, ell) % p);
                bo[j] = (uint32_t)(((uint64_t)as[j] + embv + smod(e[j], p)) % p);
                ao[j] = a[j];
            }
        }
        free(a); free(sv); free(as); free(e);
    }
}

/* CRT: residues c_i mod p_i -> the integer c in [0, q)  (textbook formula
 * c = sum_i c_i * Q_i * (Q_i^-1 mod p_i) mod q, Q_i = q / p_i). */
static u128 crt(const uint32_t* c, const uint32_t* primes, uint32_t L) {
    u128 q = prod_q(primes, L), acc = 0;
    for (uint32_t i = 0; i < L; i++) {
        u128 Qi = q / primes[i];
        uint64_t Qi_mod = (uint64_t)(Qi % primes[i]);
        uint64_t coef = mulmod(c[i], invmod(Qi_mod, primes[i]), primes[i]);
        acc = (acc + Qi * coef) % q;
    }
    return acc;
}

/* Decrypt (server step 5 of Alg. 1):
 *   u = b - a*s mod q' (CRT over the Lc limbs), m = floor((2 t u + q') / (2 q')) mod t
 * (SURVEY.md §8(c) #5).  ct layout [comp][limb<Lc][N]; out m[N]. If tv_max is
 * non-null it receives max over coefficients of |t*u - q'*m~| (m~ before mod t),
 * i.e. t times the exact noise (SURVEY.md §8(c) noise guarantee). */
void orc_decrypt_ct(uint32_t N, uint32_t Lc, const uint32_t* primes, uint32_t ell, const int8_t* s,
                    const uint32_t* ct, uint32_t* m_out, double* tv_max) {
    uint32_t* sv = (uint32_t*)malloc(4ULL * N);
    uint32_t* as = (uint32_t*)malloc(4ULL * N * Lc);
    for (uint32_t i = 0; i < Lc; i++) {
        for (uint32_t j = 0; j < N; j++) sv[j] = smod(s[j], primes[i]);
        orc_negacyclic_ntt(N, primes[i], ct + (uint64_t)(Lc + i) * N, sv, as + (uint64_t)i * N);
    }
    u128 qp = prod_q(primes, Lc), t = (u128)1 << ell;
    double mx = 0;
    uint32_t res[8];
    for (uint32_t j = 0; j < N; j++) {
        for (uint32_t i = 0; i < Lc; i++) {
            uint32_t p = primes[i];
            res[i] = (uint32_t)(((uint64_t)ct[(uint64_t)i * N + j] + p - as[(uint64_t)i * N + j]) % p);
        }
        u128 u = crt(res, primes, Lc);
        u128 mt = (2 * t * u + qp) / (2 * qp);
        m_out[j] = (uint32_t)(mt % t);
        u128 tu = t * u, qm = qp * mt;
        double d = tu >= qm ? (double)(tu - qm) : (double)(qm - tu);
        if (d > mx) mx = d;
    }
    if (tv_max) *tv_max = mx;
    free(sv); free(as);
}

/* ------------------------------------------------------------------------- */
/* COP client steps (Alg. 1)                                */
/* ------------------------------------------------------------------------- */

/* Step 2: c[alpha] = sum_beta x_{alpha,beta} (x) Enc(W_beta),
 * the scalar-ciphertext product (x) of PAPER.md:607 applied to both
 * components and every limb, summed exactly (uint128) and reduced mod p.
 * X: k x m (< t, unsigned representative).
 * Output C[alpha][comp][limb][j]  (k x 2LN). */
void orc_cop_accumulate(uint32_t N, uint32_t L, const uint32_t* primes, const uint32_t* encW,
                        const uint32_t* X, uint32_t k, uint32_t m, uint32_t* C) {
    uint64_t ncol = 2ULL * L * N;
    #pragma omp parallel
    {
        u128* acc = (u128*)malloc(sizeof(u128) * ncol);
        #pragma omp for schedule(dynamic)
        for (int64_t alpha = 0; alpha < (int64_t)k; alpha++) {
            memset(acc, 0, sizeof(u128) * ncol);
            for (uint32_t beta = 0; beta < m; beta++) {
                uint64_t x = X[(uint64_t)alpha * m + beta];
                const uint32_t* row = encW + (uint64_t)beta * ncol;
                for (uint64_t c = 0; c < ncol; c++) acc[c] += (u128)x * row[c];
            }
            for (uint64_t c = 0; c < ncol; c++) {
                uint32_t p = primes[(c / N) % L];
                C[(uint64_t)alpha * ncol + c] = (uint32_t)(acc[c] % p);
            }
        }
        free(acc);
    }
}

/* R = floor(N/n) rows per packed ciphertext (Alg. 1 step 3). */
static uint32_t rows_per_ct(uint32_t N, uint32_t n) { return N / n; }

uint32_t orc_cts_per_query(uint32_t N, uint32_t n, uint32_t kq) {
    uint32_t R = rows_per_ct(N, n);
    return (kq + R - 1) / R; /* "Pad with zeros" */
}

/* Step 3 (PAPER.md:672-679 with stride n):
 *   ct~[theta] = sum_{r<R, theta*R+r < kq} RShift(c[theta*R + r], r*n)
 * where RShift(., s) multiplies both components by X^s mod X^N+1
 * (PAPER.md:608): coefficient j moves to j+s, negated when it wraps.
 * One packed coefficient (comp, limb, J) of query-local theta. */
static uint32_t pack_coef(uint32_t N, uint32_t L, const uint32_t* primes, const uint32_t* C,
                          uint32_t n, uint32_t kq, uint32_t query, uint32_t theta,
                          uint32_t comp, uint32_t limb, uint32_t J) {
    uint32_t R = rows_per_ct(N, n), p = primes[limb];
    uint64_t ncol = 2ULL * L * N, sum = 0;
    for (uint32_t r = 0; r < R && theta * R + r < kq; r++) {
        uint64_t alpha = (uint64_t)query * kq + theta * R + r;
        /* (X^{rn} * c)[J] = c[J - rn] if J >= rn, else -c[J - rn + N] */
        uint64_t s = (uint64_t)r * n;
        const uint32_t* row = C + alpha * ncol + ((uint64_t)comp * L + limb) * N;
        uint32_t v = (J >= s) ? row[J - s] : (uint32_t)((p - row[J + N - s]) % p);
        sum = (sum + v) % p;
    }
    return (uint32_t)sum;
}

/* Mod-switch (north_star; the paper is silent):
 * iterated exact limb drop c <- round(c / p_last) for l = L-1 .. L_out,
 * computed from the definition: CRT to the integer c in [0, q_l), then
 * floor((2c + p)/(2p)) (p odd: no ties), reduced mod each remaining prime. */
static void moddown_coef(uint32_t* res, uint32_t L, uint32_t L_out, const uint32_t* primes) {
    for (uint32_t l = L; l > L_out; l--) {
        u128 c = crt(res, primes, l);
        u128 p = primes[l - 1];
        u128 d = (2 * c + p) / (2 * p);
        for (uint32_t i = 0; i < l - 1; i++) res[i] = (uint32_t)(d % primes[i]);
    }
}

/* Step 4: mask r_theta[J] uniform in Z_t
 * for every J (domain 6, index theta_global*N + J), subtracted from the b
 * component only, as Emb_{q'}(r), after the mod-switch. */
static uint32_t mask_value(uint64_t seed, uint64_t theta_global, uint32_t N, uint32_t J, uint32_t ell) {
    return uniform_t(orc_word(seed, 6, theta_global * N + J), ell);
}

/* Full client pipeline for n_queries queries of kq rows each, from the
 * unpacked C of step 2.  Output cts[query][theta][comp][limb < L_out][N]
 * and R[alpha][j] (alpha over all k = n_queries*kq rows, j < n) = Y_c. */
void orc_pack_moddown_mask_rr(uint32_t N, uint32_t L, uint32_t L_out, const uint32_t* primes, uint32_t ell,
                              const uint32_t* C, uint32_t kq, uint32_t n_queries, uint32_t n,
                              uint64_t mask_seed, const uint32_t* Z0, uint32_t* cts, uint32_t* Rout);
void orc_pack_moddown_mask(uint32_t N, uint32_t L, uint32_t L_out, const uint32_t* primes, uint32_t ell,
                           const uint32_t* C, uint32_t kq, uint32_t n_queries, uint32_t n,
                           uint64_t mask_seed, uint32_t* cts, uint32_t* Rout) {
    orc_pack_moddown_mask_rr(N, L, L_out, primes, ell, C, kq, n_queries, n, mask_seed, NULL, cts, Rout);
}

/* Same, with circuit privacy (reading 26): when Z0 is not NULL the
 * packed ciphertext tg first gets the public-key encryption of zero
 * Z0[tg][comp][limb][J] (orc_rerand_zero) added at the full modulus q, then
 * ModDown and mask as above. */
void orc_pack_moddown_mask_rr(uint32_t N, uint32_t L, uint32_t L_out, const uint32_t* primes, uint32_t ell,
                              const uint32_t* C, uint32_t kq, uint32_t n_queries, uint32_t n,
                              uint64_t mask_seed, const uint32_t* Z0, uint32_t* cts, uint32_t* Rout) {
    uint32_t R = rows_per_ct(N, n), nct = orc_cts_per_query(N, n, kq);
    u128 qp = prod_q(primes, L_out);
    #pragma omp parallel for schedule(dynamic)
    for (int64_t tg = 0; tg < (int64_t)n_queries * nct; tg++) {
        uint32_t query = (uint32_t)(tg / nct), theta = (uint32_t)(tg % nct);
        uint32_t res[8];
        for (uint32_t J = 0; J < N; J++) {
            uint32_t r = mask_value(mask_seed, (uint64_t)tg, N, J, ell);
            for (uint32_t comp = 0; comp < 2; comp++) {
                for (uint32_t i = 0; i < L; i++) {
                    res[i] = pack_coef(N, L, primes, C, n, kq, query, theta, comp, i, J);
                    if (Z0)
                        res[i] = (uint32_t)(((uint64_t)res[i] + Z0[(((uint64_t)tg * 2 + comp) * L + i) * N + J]) % primes[i]);
                }
                moddown_coef(res, L, L_out, primes);
                for (uint32_t i = 0; i < L_out; i++) {
                    uint32_t v = res[i];
                    if (comp == 0) {
                        uint32_t em = (uint32_t)(emb(qp, r, ell) % primes[i]);
                        v = (uint32_t)(((uint64_t)v + primes[i] - em) % primes[i]);
                    }
                    cts[(((uint64_t)tg * 2 + comp) * L_out + i) * N + J] = v;
                }
            }
            /* R = the mask at the valid slots: J = rho*n + j, rho < R, j < n,
             * alpha = theta*R + rho < kq  ("The client keeps r, which is R") */
            uint32_t rho = J / n, j = J % n;
            if (rho < R && theta * R + rho < kq)
                Rout[((uint64_t)query * kq + theta * R + rho) * n + j] = r;
        }
    }
}

/* Steps 2-4 end to end (client role). */
void orc_cop_matmul(uint32_t N, uint32_t L, uint32_t L_out, const uint32_t* primes, uint32_t ell,
                    const uint32_t* encW, uint32_t m, uint32_t n, const uint32_t* X, uint32_t kq,
                    uint32_t n_queries, uint64_t mask_seed, uint32_t* cts, uint32_t* Rout) {
    uint64_t k = (uint64_t)kq * n_queries;
    uint32_t* C = (uint32_t*)malloc(4ULL * k * 2 * L * N);
    orc_cop_accumulate(N, L, primes, encW, X, (uint32_t)k, m, C);
    orc_pack_moddown_mask(N, L, L_out, primes, ell, C, kq, n_queries, n, mask_seed, cts, Rout);
    free(C);
}

/* Steps 2-4 with the re-randomisation of reading 26 (Z0 from orc_rerand_zero). */
void orc_cop_matmul_rr(uint32_t N, uint32_t L, uint32_t L_out, const uint32_t* primes, uint32_t ell,
                       const uint32_t* encW, uint32_t m, uint32_t n, const uint32_t* X, uint32_t kq,
                       uint32_t n_queries, uint64_t mask_seed, const uint32_t* Z0, uint32_t* cts, uint32_t* Rout) {
    uint64_t k = (uint64_t)kq * n_queries;
    uint32_t* C = (uint32_t*)malloc(4ULL * k * 2 * L * N);
    orc_cop_accumulate(N, L, primes, encW, X, (uint32_t)k, m, C);
    orc_pack_moddown_mask_rr(N, L, L_out, primes, ell, C, kq, n_queries, n, mask_seed, Z0, cts, Rout);
    free(C);
}

/* Public key ("KeyGen. Generate the RLWE key pair (sk, pk)",
 * PAPER.md:603 encryption "under a key pk"; reading 25):
 *   a_pk[i] = uniform mod p_i (domain 7, index i N + j),  e_pk = CBD(21) (domain 8, index j),
 *   b_pk[i] = a_pk[i] * s + e_pk  mod p_i   (negacyclic product, as in Encrypt).
 * Output pk[comp b=0, a=1][limb][j]. */
void orc_keygen_pk(uint32_t N, uint32_t L, const uint32_t* primes, const int8_t* s, uint64_t seed, uint32_t* pk) {
    uint32_t* a = (uint32_t*)malloc(4ULL * N);
    uint32_t* sp = (uint32_t*)malloc(4ULL * N);
    uint32_t* as = (uint32_t*)malloc(4ULL * N);
    for (uint32_t i = 0; i < L; i++) {
        uint32_t p = primes[i];
        for (uint32_t j = 0; j < N; j++) {
            a[j] = uniform_mod(orc_word(seed, 7, (uint64_t)i * N + j), p);
            sp[j] = smod(s[j], p);
        }
        orc_negacyclic_ntt(N, p, a, sp, as);
        for (uint32_t j = 0; j < N; j++) {
            int32_t e = cbd21(orc_word(seed, 8, j));
            pk[(0 * (uint64_t)L + i) * N + j] = (uint32_t)(((uint64_t)as[j] + smod(e, p)) % p);
            pk[(1 * (uint64_t)L + i) * N + j] = a[j];
        }
    }
    free(a); free(sp); free(as);
}

/* Flooding noise f uniform in [-2^F, 2^F) (F = 0: no flooding; reading 26):
 * F <= 62: the top F + 1 bits of w0 = word(seed, 12, idx), f = (w0 >> (63 - F)) - 2^F;
 * 62 < F <= 126: the top F + 1 bits of the 128-bit V = w1 2^64 + w0 with
 * w1 = word(seed, 13, idx), f = (V >> (127 - F)) - 2^F. */
static __int128 flood(uint64_t seed, uint64_t idx, uint32_t F) {
    if (F == 0) return 0;
    uint64_t w0 = orc_word(seed, 12, idx);
    if (F <= 62) return (__int128)(w0 >> (63 - F)) - ((__int128)1 << F);
    u128 V = ((u128)orc_word(seed, 13, idx) << 64) | w0;
    return (__int128)(V >> (127 - F)) - ((__int128)1 << F);
}
static uint32_t smod128(__int128 v, uint32_t p) {
    __int128 r = v % (__int128)p;
    if (r < 0) r += p;
    return (uint32_t)r;
}

/* Circuit privacy (the client's output ciphertext must not reveal
 * X_c to the key owner; reading 26): a fresh public-key encryption of
 * zero per packed ciphertext g, at the full modulus q:
 *   v = ternary (domain 9, index g N + j), e1, e2 = CBD(21) (domains 10, 11, index g N + j),
 *   f = flooding noise in [-2^F, 2^F) (domain 12, and 13 for F > 62, index g N + j; flood()),
 *   z_b[i] = v * b_pk[i] + e1 + f,  z_a[i] = v * a_pk[i] + e2  mod p_i.
 * It decrypts to v e_pk + e1 + f - e2 s (message 0).  Output z[g][comp][limb][j]. */
void orc_rerand_zero(uint32_t N, uint32_t L, const uint32_t* primes, const uint32_t* pk, uint64_t seed,
                     uint32_t n_cts, uint32_t F, uint32_t* z) {
    #pragma omp parallel for schedule(dynamic)
    for (int64_t g = 0; g < (int64_t)n_cts; g++) {
        uint32_t* vp = (uint32_t*)malloc(4ULL * N);
        uint32_t* prod = (uint32_t*)malloc(4ULL * N);
        for (uint32_t i = 0; i < L; i++) {
            uint32_t p = primes[i];
            for (uint32_t j = 0; j < N; j++) vp[j] = smod(ternary(orc_word(seed, 9, (uint64_t)g * N + j)), p);
            for (uint32_t comp = 0; comp < 2; comp++) {
                orc_negacyclic_ntt(N, p, pk + ((uint64_t)comp * L + i) * N, vp, prod);
                for (uint32_t j = 0; j < N; j++) {
                    uint64_t idx = (uint64_t)g * N + j;
                    __int128 e = comp == 0 ? (__int128)cbd21(orc_word(seed, 10, idx)) + flood(seed, idx, F)
                                           : (__int128)cbd21(orc_word(seed, 11, idx));
                    z[(((uint64_t)g * 2 + comp) * L + i) * N + j] = (uint32_t)(((uint64_t)prod[j] + smod128(e, p)) % p);
                }
            }
        }
        free(vp); free(prod);
    }
}

/* Sampled version for workloads too large for the full oracle: for each
 * sample (query, theta, J) compute the output coefficient for both
 * components and all L_out limbs, straight from Enc(W) and X (the
 * contraction restricted to the R rows and N-shifted columns it needs).
 * out[s][comp][limb<L_out]. */
void orc_cop_matmul_sampled(uint32_t N, uint32_t L, uint32_t L_out, const uint32_t* primes, uint32_t ell,
                            const uint32_t* encW, uint32_t m, uint32_t n, const uint32_t* X, uint32_t kq,
                            uint32_t n_queries, uint64_t mask_seed, uint32_t n_samples,
                            const uint32_t* s_query, const uint32_t* s_theta, const uint32_t* s_J,
                            uint32_t* out) {
    uint32_t R = rows_per_ct(N, n), nct = orc_cts_per_query(N, n, kq);
    uint64_t ncol = 2ULL * L * N;
    u128 qp = prod_q(primes, L_out);
    #pragma omp parallel for schedule(dynamic)
    for (int64_t si = 0; si < (int64_t)n_samples; si++) {
        uint32_t query = s_query[si], theta = s_theta[si], J = s_J[si];
        uint64_t tg = (uint64_t)query * nct + theta;
        uint32_t r = mask_value(mask_seed, tg, N, J, ell);
        for (uint32_t comp = 0; comp < 2; comp++) {
            uint32_t res[8];
            for (uint32_t i = 0; i < L; i++) {
                uint32_t p = primes[i];
                uint64_t sum = 0;
                for (uint32_t rr = 0; rr < R && theta * R + rr < kq; rr++) {
                    uint64_t alpha = (uint64_t)query * kq + theta * R + rr, s = (uint64_t)rr * n;
                    uint64_t jj = (J >= s) ? J - s : J + N - s;
                    u128 acc = 0;
                    for (uint32_t beta = 0; beta < m; beta++)
                        acc += (u128)X[alpha * m + beta] * encW[(uint64_t)beta * ncol + ((uint64_t)comp * L + i) * N + jj];
                    uint32_t v = (uint32_t)(acc % p);
                    if (J < s) v = (uint32_t)((p - v) % p);
                    sum = (sum + v) % p;
                }
                res[i] = (uint32_t)sum;
            }
            moddown_coef(res, L, L_out, primes);
            for (uint32_t i = 0; i < L_out; i++) {
                uint32_t v = res[i];
                if (comp == 0) {
                    uint32_t em = (uint32_t)(emb(qp, r, ell) % primes[i]);
                    v = (uint32_t)(((uint64_t)v + primes[i] - em) % primes[i]);
                }
                out[((uint64_t)si * 2 + comp) * L_out + i] = v;
            }
        }
    }
}

/* Server step 5, decryption half: decrypt every packed
 * ciphertext and unpack Z[alpha][j] = m_theta[(alpha mod R)*n + j]
 * (inverse of the packing).  Z = (X.W - R) mod t. */
void orc_decrypt_unpack(uint32_t N, uint32_t L_out, const uint32_t* primes, uint32_t ell, const int8_t* s,
                        const uint32_t* cts, uint32_t kq, uint32_t n_queries, uint32_t n,
                        uint32_t* Z, uint32_t* mfull, double* tv_max) {
    uint32_t R = rows_per_ct(N, n), nct = orc_cts_per_query(N, n, kq);
    double mx = 0;
    #pragma omp parallel for schedule(dynamic) reduction(max:mx)
    for (int64_t tg = 0; tg < (int64_t)n_queries * nct; tg++) {
        uint32_t query = (uint32_t)(tg / nct), theta = (uint32_t)(tg % nct);
        uint32_t* mm = (uint32_t*)malloc(4ULL * N);
        double d = 0;
        orc_decrypt_ct(N, L_out, primes, ell, s, cts + (uint64_t)tg * 2 * L_out * N, mm, &d);
        if (d > mx) mx = d;
        if (mfull) memcpy(mfull + (uint64_t)tg * N, mm, 4ULL * N);
        for (uint32_t rho = 0; rho < R && theta * R + rho < kq; rho++)
            for (uint32_t j = 0; j < n; j++)
                Z[((uint64_t)query * kq + theta * R + rho) * n + j] = mm[rho * n + j];
        free(mm);
    }
    if (tv_max) *tv_max = mx;
}

/* Exact helpers exposed for the pins (same definitions as used above). */
void orc_emb(const uint32_t* primes, uint32_t L, uint32_t ell, uint64_t w, uint32_t* out) {
    u128 q = prod_q(primes, L), e = emb(q, w, ell);
    for (uint32_t i = 0; i < L; i++) out[i] = (uint32_t)(e % primes[i]);
}

void orc_moddown(uint32_t* res, uint32_t L, uint32_t L_out, const uint32_t* primes) {
    moddown_coef(res, L, L_out, primes);
}

void orc_sample_uniform_mod(uint64_t seed, uint32_t dom, uint64_t start, uint64_t count, uint32_t p, uint32_t* out) {
    for (uint64_t i = 0; i < count; i++) out[i] = uniform_mod(orc_word(seed, dom, start + i), p);
}

void orc_sample_cbd21(uint64_t seed, uint32_t dom, uint64_t start, uint64_t count, int32_t* out) {
    for (uint64_t i = 0; i < count; i++) out[i] = cbd21(orc_word(seed, dom, start + i));
}
