"""Pins for the CPU oracle (oracle/nimbus_oracle.c) against what the paper and
mathematics fix, independently of the oracle's own code:

  * worked examples printed in the paper / SPEC (tests/golden/paper_examples.json),
  * closed forms and special cases (one-hot rows, constructed ModDown inputs),
  * brute force with Python integers on tiny inputs (negacyclic products,
    X.W mod t, Miller-Rabin primality),
  * invariants (decrypt round trip, additivity, linearity, noise <= bound),
  * the survey's independent known-answer reading of the PRG/sampling contract
    (tests/golden/prg_kat.json).

Each test names the passage it pins.  CPU only (runs under -m "not gpu").
"""
import hashlib
import json
import os
import random

import numpy as np
import pytest

import nimbus_inputs as ni

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KAT = json.load(open(os.path.join(GOLD, "prg_kat.json")))
PEX = json.load(open(os.path.join(GOLD, "paper_examples.json")))
P4096 = [2147377153, 2147352577]
P8192 = [2147352577, 2147205121, 2147074049]


# ----------------------------------------------------------------- brute force
def mr_is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (bases 2..41)."""
    if n < 2:
        return False
    for sp in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41):
        if n % sp == 0:
            return n == sp
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41):
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def py_negacyclic(a, b, p):
    """Integer polynomial product, then fold X^N = -1, then mod p."""
    N = len(a)
    full = [0] * (2 * N)
    for i in range(N):
        for j in range(N):
            full[i + j] += int(a[i]) * int(b[j])
    return [(full[k] - full[k + N]) % p for k in range(N)]


def py_matmul_mod(X, W, t):
    k, m = X.shape
    n = W.shape[1]
    Xo = [[int(v) for v in row] for row in X]
    Wo = [[int(v) for v in row] for row in W]
    return np.array([[sum(Xo[a][b] * Wo[b][j] for b in range(m)) % t for j in range(n)]
                     for a in range(k)], dtype=np.uint64)


def toy_pipeline(O, N, pr, ell, L_out, k, m, n, seed, X=None, W=None, nq=1):
    L = len(pr)
    pr = np.array(pr, np.uint32)
    s = O.keygen(N, seed)
    if W is None:
        W = ni.gen_W(seed, m, n, ell)
    if X is None:
        X = ni.gen_X(seed, k * nq, m, ell)
    E = O.encrypt_rows(N, L, pr, ell, s, W, seed)
    cts, R = O.cop_matmul(N, L, L_out, pr, ell, E, X, n, k, nq, seed)
    return dict(s=s, W=W, X=X, E=E, cts=cts, R=R, pr=pr)


# ----------------------------------------------------------------- PRG / sampling
def test_prg_known_answers(oracle):
    """SURVEY.md App. B PRG contract; KAT from an independent reading."""
    seed = int(KAT["seed_cfg_C1"], 16)
    assert seed == ni.seed_cfg(1)
    for dom, vals in KAT["words"].items():
        got = [hex(int(w)) for w in oracle.words(seed, int(dom), 0, 3)]
        assert got == vals


def test_samplers_known_answers(oracle):
    seed = ni.seed_cfg(1)
    assert list(oracle.keygen(4096, seed)[:8]) == KAT["sk_0_7"]
    assert list(oracle.sample_cbd21(seed, 3, 0, 8)) == KAT["cbd_row0_0_7"]
    assert list(oracle.sample_uniform_mod(seed, 2, 0, 4, P4096[0])) == KAT["a_row0_limb0_0_3"]
    # a index = (beta*L + limb)*N + j  -> limb 1 of row 0 starts at N
    assert list(oracle.sample_uniform_mod(seed, 2, 4096, 4, P4096[1])) == KAT["a_row0_limb1_0_3"]
    assert list(ni.gen_X(seed, 1, 4, 16)[0]) == KAT["X_0_0_3_l16"]
    assert list(ni.gen_W(seed, 1, 4, 16)[0]) == KAT["W_0_0_3_l16"]
    assert list(ni.uniform_mod_t(seed, 6, 4, 16)) == KAT["mask_0_3_l16"]


def test_sampler_ranges(oracle):
    """ternary in {-1,0,1}, CBD(21) in [-21,21] with
    variance 21/2 (#6), uniform mod p below p."""
    s = oracle.keygen(1 << 15, 12345)
    vals, cnt = np.unique(s, return_counts=True)
    assert list(vals) == [-1, 0, 1] and (abs(cnt / len(s) - 1 / 3) < 0.02).all()
    e = oracle.sample_cbd21(7, 3, 0, 1 << 15).astype(np.float64)
    assert e.min() >= -21 and e.max() <= 21 and abs(e.mean()) < 0.1 and abs(e.var() - 10.5) < 0.5
    u = oracle.sample_uniform_mod(9, 2, 0, 1 << 15, P4096[0])
    assert u.max() < P4096[0] and abs(u.mean() / P4096[0] - 0.5) < 0.01


# ----------------------------------------------------------------- primes
@pytest.mark.parametrize("N,L", [(4096, 2), (8192, 3), (64, 3)])
def test_primes(oracle, N, L):
    """the L largest primes < 2^31 with p = 1 mod 2N,
    descending.  Checked with an independent Miller-Rabin scan."""
    pr = [int(p) for p in oracle.primes(N, L)]
    c = ((2 ** 31 - 2) // (2 * N)) * (2 * N) + 1
    want = []
    while len(want) < L:
        if mr_is_prime(c):
            want.append(c)
        c -= 2 * N
    assert pr == want
    if str(N) in KAT["primes"]:
        assert pr == KAT["primes"][str(N)]


# ----------------------------------------------------------------- ring
def test_negacyclic_paper_examples(oracle):
    ex = PEX["negacyclic_square"]
    p = P4096[0]
    for fn in (oracle.negacyclic_schoolbook, oracle.negacyclic_ntt):
        assert list(fn(2, p, ex["a"], ex["b"])) == ex["c"]
    sh = PEX["monomial_shift"]
    xs = [0] * 4
    xs[sh["s"]] = 1
    for fn in (oracle.negacyclic_schoolbook, oracle.negacyclic_ntt):
        c = fn(4, p, sh["a"], xs)
        assert int(c[0]) == p + sh["c_minus_q_first"] and list(c[1:]) == sh["c_rest"]


@pytest.mark.parametrize("N", [8, 16, 64])
def test_negacyclic_ntt_vs_bruteforce(oracle, N):
    rng = np.random.default_rng(N)
    for p in P4096 + P8192[1:]:
        a = rng.integers(0, p, N, dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, p, N, dtype=np.uint64).astype(np.uint32)
        want = py_negacyclic(a, b, p)
        assert list(oracle.negacyclic_schoolbook(N, p, a, b)) == want
        assert list(oracle.negacyclic_ntt(N, p, a, b)) == want


def test_negacyclic_ntt_large_invariants(oracle):
    """X^s * X^(N-s) = -1 and commutativity at N=8192 with the NTT."""
    N, p = 8192, P8192[2]
    rng = np.random.default_rng(1)
    a = rng.integers(0, p, N, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, p, N, dtype=np.uint64).astype(np.uint32)
    assert (oracle.negacyclic_ntt(N, p, a, b) == oracle.negacyclic_ntt(N, p, b, a)).all()
    s = 1234
    xs = np.zeros(N, np.uint32)
    xs[s] = 1
    xns = np.zeros(N, np.uint32)
    xns[N - s] = 1
    c = oracle.negacyclic_ntt(N, p, oracle.negacyclic_ntt(N, p, a, xs), xns)
    assert (c.astype(np.int64) == (p - a.astype(np.int64)) % p).all()
    # one coefficient against the schoolbook definition
    k = 4321
    want = (sum(int(a[i]) * int(b[k - i]) for i in range(k + 1))
            - sum(int(a[i]) * int(b[k + N - i]) for i in range(k + 1, N))) % p
    assert int(oracle.negacyclic_ntt(N, p, a, b)[k]) == want


# ----------------------------------------------------------------- embedding
def test_embedding(oracle):
    """Emb_q(w) = floor((q w + t/2)/t): the known answers,
    and the defining inequality |t Emb - q w| <= t/2 via CRT of the residues."""
    for w, want in KAT["emb_N4096_l16"].items():
        assert list(oracle.emb(np.array(P4096, np.uint32), 16, int(w))) == want
    P8192_4 = [int(v) for v in oracle.primes(8192, 4)]      # 4 limbs: q w exceeds 128 bits
    for pr, ell in ((P4096, 16), (P8192, 32), (P8192, 16), (P8192_4, 16), (P8192_4, 32)):
        q = 1
        for p in pr:
            q *= p
        t = 1 << ell
        for w in [0, 1, t // 2, t - 1] + [random.Random(ell).randrange(t) for _ in range(20)]:
            res = [int(v) for v in oracle.emb(np.array(pr, np.uint32), ell, w)]
            # CRT by Python integers
            E = sum(r * (q // p) * pow(q // p, -1, p) for r, p in zip(res, pr)) % q
            assert -t // 2 < t * E - q * w <= t // 2


# ----------------------------------------------------------------- encryption
@pytest.mark.parametrize("N,pr,ell", [(64, P4096, 16), (128, P8192, 32), (4096, P4096, 16)])
def test_encrypt_decrypt_roundtrip(oracle, N, pr, ell):
    """Dec(Enc(w_hat_beta))[j] = W[beta][j] for j<n and 0 beyond (Eq. 2,
    PAPER.md:228); the a component is the uniform sample."""
    pra = np.array(pr, np.uint32)
    L = len(pr)
    seed = 0xABCDEF ^ N
    s = oracle.keygen(N, seed)
    m, n = 3, min(N, 50)
    W = ni.gen_W(seed, m, n, ell)
    E = oracle.encrypt_rows(N, L, pra, ell, s, W, seed)
    for beta in range(m):
        assert (E[beta, 1, 0, :4] == oracle.sample_uniform_mod(seed, 2, beta * L * N, 4, pr[0])).all()
        mm, tv = oracle.decrypt_ct(N, L, pra, ell, s, E[beta])
        want = np.zeros(N, np.uint32)
        want[:n] = W[beta]
        assert (mm == want).all()
        # fresh noise: |v| <= eta + 1/2  ->  t|v| <= t*21.5
        assert tv <= 21.5 * (1 << ell)


def test_rowwise_layout_example(oracle):
    """SPEC.md:289 / PAPER.md:228: [1,2,3] at N=8 -> [1,2,3,0,0,0,0,0]."""
    ex = PEX["rowwise"]
    pr = np.array(P4096, np.uint32)
    s = oracle.keygen(8, 5)
    E = oracle.encrypt_rows(8, 2, pr, 16, s, np.array([ex["row"]], np.uint32), 5)
    mm, _ = oracle.decrypt_ct(8, 2, pr, 16, s, E[0])
    assert list(mm) == ex["encoded"]


def test_additivity(oracle):
    """Addition of ciphertexts decrypts to the sum mod t."""
    N, pr, ell = 64, np.array(P4096, np.uint32), 16
    s = oracle.keygen(N, 3)
    W = ni.gen_W(3, 2, 40, ell)
    E = oracle.encrypt_rows(N, 2, pr, ell, s, W, 3).astype(np.uint64)
    tot = ((E[0] + E[1]) % pr.astype(np.uint64)[None, :, None]).astype(np.uint32)
    mm, _ = oracle.decrypt_ct(N, 2, pr, ell, s, tot)
    assert (mm[:40] == (W[0].astype(np.uint64) + W[1]) % (1 << ell)).all()


# ----------------------------------------------------------------- COP step 2
def test_cop_onehot_row_selects_ciphertext(oracle):
    """x = e_beta (one-hot row) gives c[alpha] == Enc(W_beta) bit for bit
    (Alg. 1 step 2, with x=1 (x) ct = ct)."""
    N, pr = 64, np.array(P8192, np.uint32)
    s = oracle.keygen(N, 11)
    W = ni.gen_W(11, 9, 30, 32)
    E = oracle.encrypt_rows(N, 3, pr, 32, s, W, 11)
    X = np.zeros((9, 9), np.uint32)
    for b in range(9):
        X[b, (b * 4) % 9] = 1
    C = oracle.cop_accumulate(N, 3, pr, E, X)
    for a in range(9):
        assert (C[a] == E[(a * 4) % 9]).all()


def test_cop_bruteforce_and_linearity(oracle):
    """Each output column equals sum_beta x*E mod p (Python integers), and
    COP is linear in X modulo p."""
    N, pr = 16, np.array(P4096, np.uint32)
    s = oracle.keygen(N, 2)
    W = ni.gen_W(2, 7, 10, 16)
    E = oracle.encrypt_rows(N, 2, pr, 16, s, W, 2)
    X1 = ni.gen_X(21, 5, 7, 16)
    X2 = ni.gen_X(22, 5, 7, 16)
    C1 = oracle.cop_accumulate(N, 2, pr, E, X1)
    for a in range(5):
        for comp in range(2):
            for l in range(2):
                for j in range(N):
                    want = sum(int(X1[a, b]) * int(E[b, comp, l, j]) for b in range(7)) % int(pr[l])
                    assert int(C1[a, comp, l, j]) == want
    C2 = oracle.cop_accumulate(N, 2, pr, E, X2)
    C12 = oracle.cop_accumulate(N, 2, pr, E, X1 + X2)
    P = pr.astype(np.uint64)[None, None, :, None]
    assert (C12 == (C1.astype(np.uint64) + C2) % P).all()


def test_client_counter():
    ex = PEX["client_counter"]
    assert ni.modmacs(ex["k"], ex["m"], ex["N"], 1) == 2 * ex["per_comp_limb"]


# ----------------------------------------------------------------- packing / counts
def test_ct_counts(oracle):
    for k, n, N, want in PEX["ct_counts"]["cases"]:
        assert oracle.cts_per_query(N, n, k) == want


def test_pack_two_rows_example(oracle):
    """Fig. 4 right / SPEC.md:298: N=8, n=4, two rows -> one ciphertext
    decrypting to [a0..a3, b0..b3] once the mask is added back."""
    ex = PEX["pack_two"]
    N, n, k = ex["N"], ex["n"], ex["k"]
    pr = np.array(P4096, np.uint32)
    seed = 77
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, 3, n, 16)
    E = oracle.encrypt_rows(N, 2, pr, 16, s, W, seed)
    X = ni.gen_X(seed, k, 3, 16)
    cts, R = oracle.cop_matmul(N, 2, 1, pr, 16, E, X, n, k, 1, seed)
    assert cts.shape[:2] == (1, 1)
    _, full, _ = oracle.decrypt_unpack(N, 1, pr, 16, s, cts, k, 1, n, want_full=True)
    Y = py_matmul_mod(X, W, 1 << 16)
    mask = ni.uniform_mod_t(seed, 6, N, 16)
    got = (full[0].astype(np.uint64) + mask) % (1 << 16)
    assert list(got) == list(Y[0]) + list(Y[1])


# ----------------------------------------------------------------- ModDown
@pytest.mark.parametrize("pr,L_out", [(P4096, 1), (P8192, 2), (P8192, 1)])
def test_moddown_constructed(oracle, pr, L_out):
    """ModDown = iterated round(c / p_last).  Pin:
    c = p*y + rho with |rho| < p/2 has round(c/p) = y exactly."""
    rng = random.Random(len(pr) * 10 + L_out)
    for _ in range(200):
        # build c backwards from the answer y, one dropped prime at a time
        y = rng.randrange(1, 2 ** 28)
        c = y
        for l in range(L_out, len(pr)):
            p = pr[l]
            c = c * p + rng.randint(-(p - 1) // 2, (p - 1) // 2)
            c = max(c, 0)
        res = np.array([c % p for p in pr], np.uint32)
        got = oracle.moddown(res, L_out, np.array(pr, np.uint32))
        # expected: apply round-half-up division by integers, iterated
        want = c
        for l in range(len(pr) - 1, L_out - 1, -1):
            want = (2 * want + pr[l]) // (2 * pr[l])
        assert list(got) == [want % p for p in pr[:L_out]]
        if len(pr) - L_out == 1:
            assert want == y or c == 0


# ----------------------------------------------------------------- end to end
def _check_e2e(O, d, N, pr, ell, L_out, k, n, nq=1):
    t = 1 << ell
    Z, full, tv = O.decrypt_unpack(N, L_out, np.array(pr[:L_out], np.uint32), ell, d["s"], d["cts"],
                                   k, nq, n, want_full=True)
    Y = py_matmul_mod(d["X"], d["W"], t)
    assert (Z.astype(np.uint64) == (Y + t - d["R"]) % t).all()     # unpack(Dec) = X.W - R mod t
    # invalid slots decrypt to -r mod t
    R_ = N // n
    nct = -(-k // R_)
    for q in range(nq):
        for th in range(nct):
            tg = q * nct + th
            mask = ni.uniform_mod_t(int(d["seed"]), 6, N, ell, start=tg * N).astype(np.uint64)
            rows = min(R_, k - th * R_)
            inval = np.ones(N, bool)
            inval[: rows * n] = False
            assert (full[tg][inval] == (t - mask[inval]) % t).all()
            # R is the mask at the valid slots
            for rho in range(rows):
                assert (d["R"][q * k + th * R_ + rho] == mask[rho * n:(rho + 1) * n]).all()
    return tv / t


def noise_bound_after_moddown(N, pr, ell, L_out, m, R_eff, eta=21):
    """SURVEY.md §8(c) worst case: |v| <= R_eff*m*(t-1)*(eta+1/2) after COP and
    packing, each limb drop maps v -> v/p + (1+N)/2, the mask adds 1/2."""
    t = 1 << ell
    v = R_eff * m * (t - 1) * (eta + 0.5)
    for l in range(len(pr) - 1, L_out - 1, -1):
        v = v / pr[l] + (1 + N) / 2
    return v + 0.5


@pytest.mark.parametrize("case", [
    dict(N=64, pr=P4096, ell=16, L_out=1, k=12, m=16, n=20, nq=1),
    dict(N=64, pr=P8192, ell=32, L_out=2, k=12, m=16, n=20, nq=1),
    dict(N=64, pr=P8192, ell=16, L_out=1, k=7, m=9, n=64, nq=2),
    dict(N=128, pr=P8192, ell=32, L_out=2, k=30, m=40, n=13, nq=3),
    dict(N=256, pr=P4096, ell=16, L_out=1, k=33, m=20, n=100, nq=1),
])
def test_e2e_decrypt_equals_matmul_minus_mask(oracle, case):
    """The north-star pin: Dec(COP(X, Enc(W))) - mask = X.W mod t, brute force
    (Alg. 1 steps 4-5; SPEC.md:460 orientation), invalid slots
    = -r, R = mask, and the measured noise under the analytic bound."""
    c = case
    seed = 0x1234 + c["N"] + c["k"]
    d = toy_pipeline(oracle, c["N"], c["pr"], c["ell"], c["L_out"], c["k"], c["m"], c["n"], seed,
                     nq=c["nq"])
    d["seed"] = seed
    v = _check_e2e(oracle, d, c["N"], c["pr"], c["ell"], c["L_out"], c["k"], c["n"], c["nq"])
    R_eff = min(c["N"] // c["n"], c["k"])
    assert v <= noise_bound_after_moddown(c["N"], c["pr"], c["ell"], c["L_out"], c["m"], R_eff)


def test_e2e_exhaustive_rows_l4(oracle):
    """SPEC.md:681-style exhaustive check over Z_{2^4}: every 2-entry X row
    (256 rows) against several W, N=8, n=2 (R=4)."""
    N, ell, n, m = 8, 4, 2, 2
    X = np.array([[a, b] for a in range(16) for b in range(16)], np.uint32)
    for wseed in range(6):
        W = ni.gen_W(wseed, m, n, ell)
        d = toy_pipeline(oracle, N, P4096, ell, 1, len(X), m, n, 900 + wseed, X=X, W=W)
        d["seed"] = 900 + wseed
        _check_e2e(oracle, d, N, P4096, ell, 1, len(X), n)


def test_e2e_identity_weights(oracle):
    """W = I gives X back."""
    N, ell, m = 64, 16, 8
    W = np.eye(m, dtype=np.uint32)
    X = ni.gen_X(5, 10, m, ell)
    d = toy_pipeline(oracle, N, P4096, ell, 1, 10, m, m, 55, X=X, W=W)
    Z, _, _ = oracle.decrypt_unpack(N, 1, np.array(P4096[:1], np.uint32), ell, d["s"], d["cts"], 10, 1, m)
    assert (((Z.astype(np.uint64) + d["R"]) % (1 << ell)) == X).all()


# ----------------------------------------------------------------- server, Alg. 1 step 5
@pytest.mark.parametrize("ell", [4, 8, 12, 16, 32])
def test_plain_matmul_bruteforce(oracle, ell):
    """The server's W<X>_s mod 2^ell against Python integers, at
    full-range entries (t-1 everywhere exercises every carry) and random ones."""
    t = 1 << ell
    for k, m, n, seed in ((3, 5, 4, 1), (7, 33, 9, 2)):
        X = ni.gen_X(seed, k, m, ell)
        W = ni.gen_W(seed, m, n, ell)
        assert (oracle.plain_matmul(X, W, ell) == py_matmul_mod(X, W, t)).all()
    X = np.full((2, 40), t - 1, np.uint32)
    W = np.full((40, 3), t - 1, np.uint32)
    assert (oracle.plain_matmul(X, W, ell) == py_matmul_mod(X, W, t)).all()


@pytest.mark.parametrize("case", [
    dict(N=64, pr=P4096, ell=16, L_out=1, k=12, m=16, n=20, nq=1),
    dict(N=64, pr=P8192, ell=32, L_out=2, k=12, m=16, n=20, nq=2),
    dict(N=128, pr=P8192, ell=16, L_out=1, k=9, m=30, n=128, nq=1),
])
def test_protocol_shares_reconstruct(oracle, case):
    """Alg. 1 end to end: with X = <X>_s + <X>_c mod t, the
    server's <Y>_s = W<X>_s + Dec(...) and the client's <Y>_c = R satisfy
    <Y>_s + <Y>_c = X.W mod t (brute force with Python integers)."""
    c = case
    t = 1 << c["ell"]
    seed = 0xABC + c["N"] + c["k"]
    d = toy_pipeline(oracle, c["N"], c["pr"], c["ell"], c["L_out"], c["k"], c["m"], c["n"], seed, nq=c["nq"])
    Xc = d["X"]
    Xs = ni.gen_X(seed + 1, Xc.shape[0], c["m"], c["ell"])
    Ys = oracle.server_output(c["N"], c["L_out"], np.array(c["pr"][:c["L_out"]], np.uint32), c["ell"], d["s"],
                              d["cts"], Xs, d["W"], c["k"], c["nq"])
    X = (Xc.astype(np.uint64) + Xs) % t
    want = py_matmul_mod(X, d["W"], t)
    assert ((Ys.astype(np.uint64) + d["R"]) % t == want).all()
    assert not (Ys == want).all()          # the server's share alone is not the product


def test_toy_known_answer_digests(oracle):
    """Survey's independent reading of the whole contract, toy shape."""
    toy = KAT["toy"]
    sh = toy["shape"]
    for key, pr, ell, L_out in (("N4096_l16_Lout1", P4096, 16, 1), ("N8192_l32_Lout2", P8192, 32, 2)):
        ref = toy[key]
        seed = ni.seed_cfg(ref["cfg"])
        d = toy_pipeline(oracle, sh["N"], pr, ell, L_out, sh["k"], sh["m"], sh["n"], seed)
        assert hashlib.sha256(d["E"].tobytes()).hexdigest() == ref["enc_sha256"]
        assert hashlib.sha256(d["cts"].tobytes()).hexdigest() == ref["out_sha256"]
        assert hashlib.sha256(d["R"].tobytes()).hexdigest() == ref["R_sha256"]
        if "out_b_limb0_0_3" in ref:
            assert list(d["cts"][0, 0, 0, 0, :4]) == ref["out_b_limb0_0_3"]


def test_sampled_equals_full(oracle):
    """The sampled oracle (used at full sizes) agrees with the full oracle."""
    N, pr, ell, L_out, k, m, n, nq = 128, P8192, 32, 2, 23, 17, 40, 2
    d = toy_pipeline(oracle, N, pr, ell, L_out, k, m, n, 4242, nq=nq)
    rng = np.random.default_rng(0)
    nct = d["cts"].shape[1]
    sq = rng.integers(0, nq, 300).astype(np.uint32)
    st = rng.integers(0, nct, 300).astype(np.uint32)
    sJ = rng.integers(0, N, 300).astype(np.uint32)
    out = oracle.cop_matmul_sampled(N, 3, L_out, d["pr"], ell, d["E"], d["X"], n, k, nq, 4242, sq, st, sJ)
    for i in range(300):
        assert (out[i] == d["cts"][sq[i], st[i], :, :, sJ[i]]).all()


@pytest.mark.parametrize("N,n,k,pr", [(16, 5, 7, P4096), (64, 20, 12, P8192), (32, 32, 3, P4096)])
def test_pack_is_rshift_product(oracle, N, n, k, pr):
    """Packing = sum_r RShift(c[theta R + r], r n) where RShift multiplies by
    the monomial X^{r n} (App. B.1; stride n).
    Pinned against the schoolbook negacyclic product with Python integers on
    arbitrary unpacked inputs, with L_out = L (no mod-switch): the a component
    is unmasked; the b component carries -Emb_q(r)."""
    L, ell = len(pr), 16
    pra = np.array(pr, np.uint32)
    rng = np.random.default_rng(N + n + k)
    Cu = np.stack([np.stack([np.stack([rng.integers(0, p, N, dtype=np.uint64) for p in pr])
                             for _ in range(2)]) for _ in range(k)]).astype(np.uint32)
    cts, R = oracle.pack_moddown_mask(N, L, L, pra, ell, Cu, k, 1, n, 99)
    Rr = N // n
    for th in range(cts.shape[1]):
        mask = ni.uniform_mod_t(99, 6, N, ell, start=th * N)
        for comp in range(2):
            for l, p in enumerate(pr):
                acc = [0] * N
                for r in range(Rr):
                    if th * Rr + r >= k:
                        break
                    mono = [0] * N
                    mono[r * n] = 1
                    prod = py_negacyclic(Cu[th * Rr + r, comp, l], mono, p)
                    acc = [(x + y) % p for x, y in zip(acc, prod)]
                if comp == 0:
                    emb = [int(oracle.emb(pra, ell, int(w))[l]) for w in mask]
                    acc = [(x - e) % p for x, e in zip(acc, emb)]
                assert list(cts[0, th, comp, l]) == acc


# ----------------------------------------------------------------- wide oracle (ell = 64, q > 2^128)
def test_wide_oracle_equals_c_oracle(oracle):
    """The Python-integer oracle (oracle/wide.py) follows the same steps as the C
    oracle; where both apply (ell = 16, 2 limbs) they give the same bytes for
    Enc(W), the output ciphertexts, R and the decrypted Z."""
    from oracle import wide
    N, pr, ell, L_out, k, m, n = 64, P4096, 16, 1, 7, 9, 20
    seed = 0xBEEF
    d = toy_pipeline(oracle, N, pr, ell, L_out, k, m, n, seed)
    Ew = wide.encrypt_rows(N, 2, np.array(pr, np.uint32), ell, d["s"], d["W"], seed)
    assert (Ew == d["E"]).all()
    cts, R = wide.cop_matmul(N, 2, L_out, pr, ell, d["E"], d["X"], n, k, 1, seed)
    assert (cts == d["cts"]).all() and (R == d["R"]).all()
    Zw, _ = wide.decrypt_unpack(N, L_out, pr, ell, d["s"], cts, k, 1, n)
    Zc, _, _ = oracle.decrypt_unpack(N, L_out, np.array(pr[:L_out], np.uint32), ell, d["s"], d["cts"], k, 1, n)
    assert (Zw == Zc).all()


@pytest.mark.parametrize("case", [dict(N=64, L=5, L_out=3, k=6, m=5, n=20, nq=1),
                                  dict(N=128, L=5, L_out=3, k=5, m=12, n=50, nq=2)])
def test_wide_e2e_ell64(oracle, case):
    """The paper's ell = 64 with 5 limbs (q ~ 2^155) and a 3-limb
    output: Dec - mask = X.W mod 2^64 by Python-integer brute force, round trip of
    Enc(W) rows (Eq. 2), invalid slots = -r."""
    from oracle import wide
    c = case
    N, L, L_out, ell = c["N"], c["L"], c["L_out"], 64
    pr = [int(p) for p in oracle.primes(N, L)]
    t = 1 << ell
    seed = 0x64 + N
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, c["m"], c["n"], ell)
    X = ni.gen_X(seed, c["k"] * c["nq"], c["m"], ell)
    assert W.dtype == np.uint64 and int(W.max()) >= (1 << 62)    # full-width entries
    E = wide.encrypt_rows(N, L, pr, ell, s, W, seed)
    # Dec(Enc(w_hat_beta)) = W[beta] then zeros (row-wise encoding)
    for beta in range(c["m"]):
        ct = E[beta][None, None]                                  # as one packed ct with all L limbs
        Zr, full = wide.decrypt_unpack(N, L, pr, ell, s, ct, 1, 1, N)
        assert [int(v) for v in full[0][:c["n"]]] == [int(v) for v in W[beta]]
        assert not full[0][c["n"]:].any()
    cts, R = wide.cop_matmul(N, L, L_out, pr, ell, E, X, c["n"], c["k"], c["nq"], seed)
    Z, full = wide.decrypt_unpack(N, L_out, pr, ell, s, cts, c["k"], c["nq"], c["n"])
    Y = py_matmul_mod(X, W, t)
    assert all(int(Z[a, j]) == (int(Y[a, j]) - int(R[a, j])) % t for a in range(Z.shape[0]) for j in range(c["n"]))
    R_ = N // c["n"]
    nct = -(-c["k"] // R_)
    for tg in range(c["nq"] * nct):
        th = tg % nct
        rows = min(R_, c["k"] - th * R_)
        mask = oracle.words(seed, 6, tg * N, N)
        for J in range(rows * c["n"], N):
            assert int(full[tg, J]) == (t - int(mask[J])) % t


# ----------------------------------------------------------------- server step 5 at ell = 64
def test_plain_matmul64_bruteforce(oracle):
    """The server's W<X>_s mod 2^64 (PAPER.md:681 at the paper's t) against Python
    integers: random full-width entries and all-(2^64 - 1) entries (every carry)."""
    from oracle import wide
    t = 1 << 64
    for k, m, n, seed in ((3, 5, 4, 1), (6, 37, 9, 2)):
        X = ni.gen_X(seed, k, m, 64)
        W = ni.gen_W(seed, m, n, 64)
        got = wide.plain_matmul64(X, W)
        want = py_matmul_mod(X, W, t)
        assert all(int(got[a, j]) == int(want[a, j]) for a in range(k) for j in range(n))
    X = np.full((2, 40), t - 1, np.uint64)
    W = np.full((40, 3), t - 1, np.uint64)
    assert all(int(v) == (40 * (t - 1) ** 2) % t for v in wide.plain_matmul64(X, W).ravel())


def test_server_output_ell64_reconstructs(oracle):
    """Alg. 1 end to end at t = 2^64: with X = <X>_s + <X>_c mod 2^64 the
    server's <Y>_s (wide oracle: decrypt + unpack + its own product) and the client's R satisfy
    <Y>_s + R = X.W mod 2^64 by Python integers, and <Y>_s alone is not the product."""
    from oracle import wide
    N, L, L_out, ell, k, m, n, nq = 64, 5, 3, 64, 6, 7, 20, 1
    t = 1 << ell
    pr = [int(p) for p in oracle.primes(N, L)]
    seed = 0x5E64
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, m, n, ell)
    Xc = ni.gen_X(seed, k, m, ell)
    Xs = ni.gen_X(seed + 1, k, m, ell)
    E = wide.encrypt_rows(N, L, pr, ell, s, W, seed)
    cts, R = wide.cop_matmul(N, L, L_out, pr, ell, E, Xc, n, k, nq, seed)
    Ys = wide.server_output(N, L_out, pr, ell, s, cts, Xs, W, k, nq)
    X = [[(int(Xc[a, b]) + int(Xs[a, b])) % t for b in range(m)] for a in range(k)]
    want = [[sum(X[a][b] * int(W[b, j]) for b in range(m)) % t for j in range(n)] for a in range(k)]
    assert all((int(Ys[a, j]) + int(R[a, j])) % t == want[a][j] for a in range(k) for j in range(n))
    assert any(int(Ys[a, j]) != want[a][j] for a in range(k) for j in range(n))


def test_wide_sampled_equals_full(oracle):
    """wide.cop_matmul_sampled (the full-size check of the ell = 64 bytes) returns exactly the
    coefficients wide.cop_matmul computes, on every slot of a small two-query case (incl. wrapped
    shifts, the ragged last packed ciphertext and invalid slots)."""
    from oracle import wide
    N, L, L_out, ell, k, m, n, nq = 64, 5, 3, 64, 7, 5, 20, 2
    pr = [int(p) for p in oracle.primes(N, L)]
    seed = 0x5A3
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, m, n, ell)
    X = ni.gen_X(seed, k * nq, m, ell)
    E = wide.encrypt_rows(N, L, pr, ell, s, W, seed)
    cts, _ = wide.cop_matmul(N, L, L_out, pr, ell, E, X, n, k, nq, seed)
    nct = cts.shape[1]
    sq, st, sJ = np.meshgrid(np.arange(nq), np.arange(nct), np.arange(N), indexing="ij")
    got = wide.cop_matmul_sampled(N, L, L_out, pr, ell, E, X, n, k, nq, seed, sq.ravel(), st.ravel(), sJ.ravel())
    assert (got == cts.transpose(0, 1, 4, 2, 3).reshape(-1, 2, L_out)).all()
