"""Oracle for parameter sets beyond the C oracle's 128-bit integers: the
paper's ell = 64 with q = 5 x 31-bit primes (~2^155).

TEST INFRASTRUCTURE ONLY (same rule as oracle.py): imported by tests/ and the
bench's cpu_baseline leg, never by the product package.

Every step follows the same passage as its C-oracle counterpart, in the same
order, with Python integers where q or 2 t u exceed 128 bits; the
per-limb pieces reuse the C oracle's own primitives (PRG and samplers, and
the negacyclic product mod p_i), which are pinned in test_oracle_pins.py.
Small sizes only (the contraction is a Python/numpy loop).
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def _q(pr) -> int:
    q = 1
    for p in pr:
        q *= int(p)
    return q


def emb(q: int, w: int, ell: int) -> int:
    """Emb_q(w) = floor((q w + t/2) / t) (§2.1)."""
    t = 1 << ell
    return (q * w + t // 2) // t


def encrypt_rows(N, L, pr, ell, s, W, seed) -> np.ndarray:
    """Alg. 1 step 1, row-wise encoding Eq. 2:
    for row beta and limb i, a_i uniform mod p_i (domain 2, index (beta L + i) N + j),
    e = CBD(21) (domain 3, index beta N + j), b_i = a_i s + Emb_q(w_hat) + e mod p_i.
    Output [beta][comp b=0, a=1][limb][j] uint32."""
    pr = [int(p) for p in pr]
    q = _q(pr)
    W = np.asarray(W, dtype=np.uint64)
    m, n = W.shape
    out = np.empty((m, 2, L, N), np.uint32)
    sps = [np.array([int(x) % p for x in s], np.uint32) for p in pr]
    for beta in range(m):
        e = O.sample_cbd21(seed, 3, beta * N, N).astype(np.int64)
        # w_hat[j] = W[beta][j] for j < n, else 0 (Emb_q(0) = 0): only the first n slots need Emb
        embs = [emb(q, int(W[beta, j]), ell) for j in range(n)]
        for i, p in enumerate(pr):
            a = O.sample_uniform_mod(seed, 2, (beta * L + i) * N, N, p)
            a_s = O.negacyclic_ntt(N, p, a, sps[i]).astype(np.int64)
            em = np.zeros(N, np.int64)
            em[:n] = np.array([x % p for x in embs], np.int64)
            out[beta, 0, i] = ((a_s + em + e) % p).astype(np.uint32)
            out[beta, 1, i] = a
    return out


def _moddown(c: list, pr: list, L_out: int) -> list:
    """Iterated exact limb drop c <- round(c / p_last) = floor((2c + p)/(2p)) on the
    CRT integer, smallest prime first."""
    res = list(c)
    for l in range(len(pr), L_out, -1):
        ql = _q(pr[:l])
        x = 0
        for i in range(l):                       # CRT to the integer in [0, q_l)
            Qi = ql // pr[i]
            x += res[i] * Qi * pow(Qi, -1, pr[i])
        x %= ql
        p = pr[l - 1]
        d = (2 * x + p) // (2 * p)
        res = [d % pr[i] for i in range(l - 1)]
    return res


def cop_matmul(N, L, L_out, pr, ell, E, X, n, kq, nq, seed, Z0=None):
    """Alg. 1 steps 2-4: c[alpha] = sum_beta x (x) Enc(W_beta)
    per limb mod p_i; RShift packing with stride n; ModDown to
    L_out limbs; mask r_theta[J] = word(seed, 6, tg N + J) >> (64 - ell) subtracted
    from b as Emb_q'(r).  Z0 (optional, [nq*nct][2][L][N]): public-key encryptions of
    zero added before ModDown (circuit privacy, reading 26).
    Returns (cts [nq][nct][2][L_out][N] uint32, R [k][n] uint64)."""
    pr = [int(p) for p in pr]
    t = 1 << ell
    X = np.asarray(X, dtype=np.uint64)
    k, m = X.shape
    E = np.asarray(E, dtype=np.uint64)
    # step 2: unpacked C[alpha][comp][limb][j]
    C = np.zeros((k, 2, L, N), dtype=object)
    for i, p in enumerate(pr):
        Xp = np.array([[int(x) % p for x in row] for row in X], dtype=np.uint64)   # scalar mod p_i
        acc = np.zeros((k, 2, N), dtype=np.uint64)
        for beta in range(m):
            acc = (acc + (Xp[:, beta][:, None, None] * E[beta, :, i, :][None]) % np.uint64(p)) % np.uint64(p)
        C[:, :, i, :] = acc
    R_ = N // n
    nct = -(-kq // R_)
    qo = _q(pr[:L_out])
    cts = np.zeros((nq, nct, 2, L_out, N), np.uint32)
    R = np.zeros((nq * kq, n), np.uint64)
    for q_ in range(nq):
        for th in range(nct):
            tg = q_ * nct + th
            rows = min(R_, kq - th * R_)
            mask = O.words(seed, 6, tg * N, N) >> np.uint64(64 - ell) if ell < 64 else O.words(seed, 6, tg * N, N)
            for comp in range(2):
                for J in range(N):
                    c = []
                    for i, p in enumerate(pr):
                        v = 0
                        for r in range(rows):           # RShift: X^(r n) c[theta R + r]
                            sh = r * n
                            val = int(C[q_ * kq + th * R_ + r, comp, i, (J - sh) % N])
                            v += val if J >= sh else p - val
                        if Z0 is not None:
                            v += int(Z0[tg, comp, i, J])
                        c.append(v % p)
                    c = _moddown(c, pr, L_out)
                    if comp == 0:
                        em = emb(qo, int(mask[J]), ell)
                        c = [(c[i] - em) % pr[i] for i in range(L_out)]
                    cts[q_, th, comp, :, J] = c
            for rho in range(rows):
                R[q_ * kq + th * R_ + rho] = mask[rho * n:(rho + 1) * n]
    return cts, R


def decrypt_unpack(N, L_out, pr, ell, s, cts, kq, nq, n):
    """Server step 5 decryption: u = b - a s mod q' (per limb
    with the C oracle's negacyclic product, CRT in Python integers),
    m = floor((2 t u + q') / (2 q')) mod t; unpack
    Z[alpha][j] = m_theta[(alpha mod R) n + j].  Returns (Z uint64, full slots)."""
    pr = [int(p) for p in pr[:L_out]]
    t = 1 << ell
    qo = _q(pr)
    cts = np.asarray(cts, dtype=np.uint32)
    nct = cts.shape[1]
    R_ = N // n
    Z = np.zeros((nq * kq, n), np.uint64)
    full = np.zeros((nq * nct, N), np.uint64)
    for q_ in range(nq):
        for th in range(nct):
            us = []
            for i, p in enumerate(pr):
                sp = np.array([int(x) % p for x in s], np.uint32)
                a_s = O.negacyclic_ntt(N, p, cts[q_, th, 1, i], sp)
                us.append([(int(cts[q_, th, 0, i, j]) - int(a_s[j])) % p for j in range(N)])
            ms = []
            for j in range(N):
                u = 0
                for i, p in enumerate(pr):
                    Qi = qo // p
                    u += us[i][j] * Qi * pow(Qi, -1, p)
                u %= qo
                ms.append(((2 * t * u + qo) // (2 * qo)) % t)
            full[q_ * nct + th] = np.array(ms, dtype=np.uint64)
            rows = min(R_, kq - th * R_)
            for rho in range(rows):
                Z[q_ * kq + th * R_ + rho] = full[q_ * nct + th][rho * n:(rho + 1) * n]
    return Z, full


def plain_matmul64(X, W) -> np.ndarray:
    """The server's W<X>_s at the paper's t = 2^64 (Alg. 1 step 5; ell = 64,
    PAPER.md:402): the textbook product of the uint64 matrices, whose wrap-around IS the
    reduction mod 2^64 (Y = X.W, SURVEY.md §8(c) #10 orientation)."""
    X = np.ascontiguousarray(X, dtype=np.uint64)
    W = np.ascontiguousarray(W, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return X @ W


def server_output(N, L_out, pr, ell, s, cts, Xs, W, kq, nq) -> np.ndarray:
    """Alg. 1 step 5 at ell = 64: <Y>_s = W<X>_s + (W<X>_c - R) mod 2^64, the
    second term the server's decryption + unpack of the client's ciphertexts (decrypt_unpack)."""
    assert ell == 64
    Z, _ = decrypt_unpack(N, L_out, pr, ell, s, cts, kq, nq, np.asarray(W).shape[1])
    with np.errstate(over="ignore"):
        return plain_matmul64(Xs, W) + Z


def cop_matmul_sampled(N, L, L_out, pr, ell, E, X, n, kq, nq, seed, s_query, s_theta, s_J) -> np.ndarray:
    """cop_matmul restricted to sampled output coefficients (query, theta, J), for sizes the full
    oracle cannot run: the same steps (per-limb contraction mod p_i of the rows theta R + r and the
    columns (J - r n) mod N RShift packing reads, ModDown on the CRT integer, the mask Emb_q'(r)).
    Returns out[sample][comp][limb < L_out] uint32."""
    pr = [int(p) for p in pr]
    t = 1 << ell
    X = np.asarray(X, dtype=np.uint64)
    E = np.asarray(E)
    R_ = N // n
    nct = -(-kq // R_)
    qo = _q(pr[:L_out])
    out = np.zeros((len(s_query), 2, L_out), np.uint32)
    for si, (q_, th, J) in enumerate(zip(s_query, s_theta, s_J)):
        q_, th, J = int(q_), int(th), int(J)
        tg = q_ * nct + th
        rows = min(R_, kq - th * R_)
        w = int(O.words(seed, 6, tg * N + J, 1)[0])
        r_mask = w >> (64 - ell) if ell < 64 else w
        for comp in range(2):
            c = []
            for i, p in enumerate(pr):
                v = 0
                for r in range(rows):            # RShift: X^(r n) c[theta R + r]
                    sh = r * n
                    col = (J - sh) % N
                    xs = np.array([int(x) % p for x in X[q_ * kq + th * R_ + r]], dtype=object)
                    es = E[:, comp, i, col].astype(object)
                    val = int((xs * es).sum()) % p
                    v += val if J >= sh else p - val
                c.append(v % p)
            c = _moddown(c, pr, L_out)
            if comp == 0:
                em = emb(qo, r_mask, ell)
                c = [(c[i] - em) % pr[i] for i in range(L_out)]
            out[si, comp] = c
    return out
