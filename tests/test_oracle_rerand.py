"""Pins for the oracle's public key and circuit-privacy re-randomisation
(oracle/nimbus_oracle.c orc_keygen_pk, orc_rerand_zero, orc_cop_matmul_rr;
DESIGN.md readings 25-26; PAPER.md:602-603 KeyGen (sk, pk) / encryption under
pk, PAPER.md:645 circuit privacy of the client's output ciphertext).

Independent of the oracle's own code: decryption identities checked with
Python-integer negacyclic products over Z (no NTT, no modulus until the end),
the protocol identity Dec - mask = X.W mod t by brute force, and the noise
bound.  CPU only.
"""
import numpy as np
import pytest

import nimbus_inputs as ni
from test_oracle_pins import P4096, P8192, py_matmul_mod, py_negacyclic


def negacyclic_Z(a, b):
    """Integer negacyclic product over Z (X^N = -1), no modulus."""
    N = len(a)
    full = [0] * (2 * N)
    for i in range(N):
        ai = int(a[i])
        if ai:
            for j in range(N):
                full[i + j] += ai * int(b[j])
    return [full[k] - full[k + N] for k in range(N)]


def centered(x, p):
    x %= p
    return x - p if x > p // 2 else x


def ternary_words(O, seed, dom, start, N):
    """App. B ternary sampler: floor(w * 3 / 2^64) - 1."""
    return [(int(w) * 3 >> 64) - 1 for w in O.words(seed, dom, start, N)]


def flood_words(O, seed, start, N, F):
    """Reading 26: f uniform in [-2^F, 2^F), the top F + 1 bits of w0 = word(seed, 12, i) (F <= 62)
    or of the 128-bit w1 2^64 + w0 with w1 = word(seed, 13, i) (62 < F <= 126); none when F = 0."""
    if F == 0:
        return [0] * N
    w0 = [int(w) for w in O.words(seed, 12, start, N)]
    if F <= 62:
        return [(w >> (63 - F)) - (1 << F) for w in w0]
    w1 = [int(w) for w in O.words(seed, 13, start, N)]
    return [(((hi << 64) | lo) >> (127 - F)) - (1 << F) for hi, lo in zip(w1, w0)]


@pytest.mark.parametrize("N,pr", [(64, P4096), (64, P8192), (128, P8192)])
def test_public_key_decrypts_to_cbd_noise(oracle, N, pr):
    """pk = (b, a) with b - a s = e_pk exactly (PAPER.md:602 KeyGen; reading 25):
    the same small integer polynomial in every limb, |e| <= 21, equal to the
    CBD(21) draw of domain 8; a is uniform mod p_i (not small)."""
    L = len(pr)
    seed = 0x9C + N
    s = oracle.keygen(N, seed)
    pk = oracle.keygen_pk(N, L, np.array(pr, np.uint32), s, seed)
    e_pk = oracle.sample_cbd21(seed, 8, 0, N).astype(np.int64)
    assert np.abs(e_pk).max() <= 21 and np.abs(e_pk).max() > 0
    for i, p in enumerate(pr):
        a, b = pk[1, i], pk[0, i]
        as_ = py_negacyclic(a, [int(v) % p for v in s], p)
        e = [centered(int(b[j]) - as_[j], p) for j in range(N)]
        assert e == [int(v) for v in e_pk]
        assert int(a.max()) > p // 2                     # uniform, not small
    # a_pk differs between limbs (independent draws, index i N + j)
    assert (pk[1, 0] != pk[1, 1] % pr[0]).any()


@pytest.mark.parametrize("F", [0, 20, 80])
def test_zero_encryption_noise_is_exact(oracle, F):
    """z = (v b_pk + e1 + f, v a_pk + e2) decrypts to exactly
    v e_pk + e1 + f - e2 s over Z (reading 26), the same integer in every limb,
    message 0 at the full modulus."""
    N, pr = 64, P8192
    L, seed, ell = len(pr), 0xA11CE, 32
    s = oracle.keygen(N, seed)
    pk = oracle.keygen_pk(N, L, np.array(pr, np.uint32), s, seed)
    e_pk = [int(v) for v in oracle.sample_cbd21(seed, 8, 0, N)]
    rseed = 0x5EED
    n_cts = 3
    z = oracle.rerand_zero(N, L, np.array(pr, np.uint32), pk, rseed, n_cts, F)
    for g in range(n_cts):
        v = ternary_words(oracle, rseed, 9, g * N, N)
        e1 = [int(x) for x in oracle.sample_cbd21(rseed, 10, g * N, N)]
        e2 = [int(x) for x in oracle.sample_cbd21(rseed, 11, g * N, N)]
        f = flood_words(oracle, rseed, g * N, N, F)
        ve = negacyclic_Z(v, e_pk)
        e2s = negacyclic_Z(e2, [int(x) for x in s])
        want = [ve[j] + e1[j] + f[j] - e2s[j] for j in range(N)]
        assert max(abs(w) for w in want) <= 42 * N + 21 + (1 << F)
        res = []
        for i, p in enumerate(pr):
            b, a = z[g, 0, i], z[g, 1, i]
            as_ = py_negacyclic(a, [int(x) % p for x in s], p)
            res.append([(int(b[j]) - as_[j]) % p for j in range(N)])
            assert [centered(r, p) for r in res[-1]] == [centered(w, p) for w in want]
        # one integer in every limb: CRT over q = prod p_i (> 2^92 > 2 |noise|) recovers it exactly
        q = 1
        for p in pr:
            q *= p
        crt = [centered(sum(res[i][j] * (q // p) * pow(q // p, -1, p) for i, p in enumerate(pr)), q)
               for j in range(N)]
        assert crt == want
        if F <= 62:     # the C oracle's decryption needs |noise| < q / (2 t) (q ~ 2^93, t = 2^32)
            m = oracle.decrypt_ct(N, L, np.array(pr, np.uint32), ell, s, z[g])[0]
            assert not np.asarray(m).any()
    if F:
        assert any(abs(x) > 42 * N + 21 for x in want)  # the flooding term is really there


def noise_bound_rr(N, pr, ell, L_out, m, R_eff, F, eta=21):
    """Worst case with the zero encryption added before ModDown: the COP bound
    R m (t-1)(eta+1/2) plus |v e_pk + e1 + f - e2 s| <= 2 eta N + eta + 2^F; each
    limb drop v -> v/p + (1+N)/2; the mask adds 1/2."""
    t = 1 << ell
    v = R_eff * m * (t - 1) * (eta + 0.5) + 2 * eta * N + eta + (1 << F if F else 0)
    for l in range(len(pr) - 1, L_out - 1, -1):
        v = v / pr[l] + (1 + N) / 2
    return v + 0.5


def max_flood_bits(N, pr, ell, L_out, m, R_eff):
    q_out = 1
    for p in pr[:L_out]:
        q_out *= p
    best = 0
    for F in range(1, 127):
        if noise_bound_rr(N, pr, ell, L_out, m, R_eff, F) < q_out / (2 * (1 << ell)):
            best = F
    return best


@pytest.mark.parametrize("case", [
    dict(N=128, pr=P8192, ell=32, L_out=2, k=30, m=40, n=13, nq=2),
    dict(N=256, pr=P4096, ell=16, L_out=1, k=33, m=20, n=100, nq=1),
    dict(N=64, pr=P8192, ell=16, L_out=1, k=7, m=9, n=64, nq=2),
])
def test_rerandomised_output_decrypts_to_the_same_shares(oracle, case):
    """Circuit privacy does not change the protocol's result (PAPER.md:645,
    680-681): with the largest flooding the bound allows, Dec - mask is still
    X.W mod t by brute force, the mask R is unchanged, and the a component (the
    part that would let the key owner solve for X_c) is a different,
    re-randomised polynomial.  With flooding far past the bound, decryption
    fails -- the bound is what keeps it exact."""
    c = case
    N, pr, ell, L_out = c["N"], c["pr"], c["ell"], c["L_out"]
    L, t = len(pr), 1 << c["ell"]
    seed = 0x77 + N
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, c["m"], c["n"], ell)
    X = ni.gen_X(seed, c["k"] * c["nq"], c["m"], ell)
    E = oracle.encrypt_rows(N, L, np.array(pr, np.uint32), ell, s, W, seed)
    cts0, R0 = oracle.cop_matmul(N, L, L_out, np.array(pr, np.uint32), ell, E, X, c["n"], c["k"], c["nq"], seed)
    R_eff = min(N // c["n"], c["k"])
    F = max_flood_bits(N, pr, ell, L_out, c["m"], R_eff)
    assert F >= 8
    pk = oracle.keygen_pk(N, L, np.array(pr, np.uint32), s, seed ^ 0xF00)
    nct = oracle.cts_per_query(N, c["n"], c["k"]) * c["nq"]
    z = oracle.rerand_zero(N, L, np.array(pr, np.uint32), pk, seed ^ 0xABC, nct, F)
    cts, R = oracle.cop_matmul_rr(N, L, L_out, np.array(pr, np.uint32), ell, E, X, c["n"], c["k"], c["nq"],
                                  seed, z)
    assert (R == R0).all()
    Z, _, tv = oracle.decrypt_unpack(N, L_out, np.array(pr[:L_out], np.uint32), ell, s, cts, c["k"], c["nq"],
                                     c["n"])
    Y = py_matmul_mod(X, W, t)
    assert (Z.astype(np.uint64) == (Y + t - R) % t).all()
    assert tv / t <= noise_bound_rr(N, pr, ell, L_out, c["m"], R_eff, F)
    a0, a1 = cts0[:, :, 1], cts[:, :, 1]
    assert (a0 != a1).mean() > 0.99
    # 4 bits past the bound: wrong plaintexts
    zbig = oracle.rerand_zero(N, L, np.array(pr, np.uint32), pk, seed ^ 0xABC, nct, F + 4)
    cbig, _ = oracle.cop_matmul_rr(N, L, L_out, np.array(pr, np.uint32), ell, E, X, c["n"], c["k"], c["nq"],
                                   seed, zbig)
    Zb, _, _ = oracle.decrypt_unpack(N, L_out, np.array(pr[:L_out], np.uint32), ell, s, cbig, c["k"], c["nq"],
                                     c["n"])
    assert (Zb.astype(np.uint64) != (Y + t - R) % t).mean() > 0.5


def test_statistical_flooding_parameter_set(oracle):
    """The shipped circuit-privacy parameter set (reading 26): one more limb (L = 3,
    L_out = 1, ell = 16) lets the flooding noise exceed the worst-case COP noise
    R m (t-1)(eta + 1/2) by >= 40 bits -- statistical smudging -- and the output
    still decrypts exactly to X.W - R mod t (brute force)."""
    N, ell, L_out, L = 256, 16, 1, 3
    pr = [int(p) for p in oracle.primes(N, L)]
    k, m, n = 12, 64, 100
    t = 1 << ell
    seed = 0xF10D
    R_eff = min(N // n, k)
    F = max_flood_bits(N, pr, ell, L_out, m, R_eff)
    cop = R_eff * m * (t - 1) * 21.5
    assert F - np.log2(cop) >= 40, (F, np.log2(cop))
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, m, n, ell)
    X = ni.gen_X(seed, k, m, ell)
    E = oracle.encrypt_rows(N, L, np.array(pr, np.uint32), ell, s, W, seed)
    pk = oracle.keygen_pk(N, L, np.array(pr, np.uint32), s, seed + 1)
    nct = oracle.cts_per_query(N, n, k)
    z = oracle.rerand_zero(N, L, np.array(pr, np.uint32), pk, seed + 2, nct, F)
    cts, R = oracle.cop_matmul_rr(N, L, L_out, np.array(pr, np.uint32), ell, E, X, n, k, 1, seed, z)
    Z, _, tv = oracle.decrypt_unpack(N, L_out, np.array(pr[:L_out], np.uint32), ell, s, cts, k, 1, n)
    Y = py_matmul_mod(X, W, t)
    assert (Z.astype(np.uint64) == (Y + t - R) % t).all()
    # the flooding term dominates the zero encryptions' noise (|f| up to 2^F)
    f = flood_words(oracle, seed + 2, 0, N, F)
    assert max(abs(x) for x in f) > 2 ** (F - 2)


def test_rerandomised_ell64_wide_oracle(oracle):
    """The paper's ell = 64 with 5 limbs: the Python-integer oracle with the zero
    encryptions added before ModDown still decrypts to X.W - R mod 2^64."""
    from oracle import wide
    N, L, L_out, ell, k, m, n = 64, 5, 3, 64, 6, 5, 20
    pr = [int(p) for p in oracle.primes(N, L)]
    t = 1 << ell
    seed = 0x6464
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, m, n, ell)
    X = ni.gen_X(seed, k, m, ell)
    E = wide.encrypt_rows(N, L, pr, ell, s, W, seed)
    pk = oracle.keygen_pk(N, L, np.array(pr, np.uint32), s, seed + 1)
    nct = -(-k // (N // n))
    z = oracle.rerand_zero(N, L, np.array(pr, np.uint32), pk, seed + 2, nct, 40)
    cts, R = wide.cop_matmul(N, L, L_out, pr, ell, E, X, n, k, 1, seed, Z0=z.reshape(nct, 2, L, N))
    Z, _ = wide.decrypt_unpack(N, L_out, pr, ell, s, cts, k, 1, n)
    Y = py_matmul_mod(X, W, t)
    assert (Z.astype(object) == (Y.astype(object) + t - R.astype(object)) % t).all()
    cts0, _ = wide.cop_matmul(N, L, L_out, pr, ell, E, X, n, k, 1, seed)
    assert (cts0[:, :, 1] != cts[:, :, 1]).mean() > 0.99
