"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle,
element by element on the same seeded inputs, plus properties that hold at any
size (decryption of every packed ciphertext equals X.W - R mod t, invalid slots
equal -r).  Bit-exact is the bar everywhere: the whole path is integer arithmetic
(SURVEY.md §8(c) "Plain definition of the result").

Sizes: full oracle comparison where the oracle finishes in seconds (toy, C1,
C2, C3, ragged multi-tile shapes); at C4/C5 sizes, full Enc(W) comparison plus
sampled output coefficients from the oracle, plus the exact decryption property
over every output.
"""
import os
import numpy as np
import pytest
import torch

import nimbus_inputs as ni

pytestmark = pytest.mark.gpu

P4096 = [2147377153, 2147352577]
P8192 = [2147352577, 2147205121, 2147074049]
DEV = "cuda:0"


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_15707_b200 import nimbus
    nimbus.lib()
    return nimbus


def u32(t):
    from paper_2411_15707_b200 import nimbus
    return nimbus.to_numpy_u32(t)


def dev_u32(a):
    from paper_2411_15707_b200 import nimbus
    return nimbus.from_numpy_u32(a, DEV)


def matmul_mod_t(X, W, ell):
    """X.W mod 2^ell with uint64 wrap-around arithmetic (exact mod 2^64)."""
    with np.errstate(over="ignore"):
        Y = X.astype(np.uint64) @ W.astype(np.uint64)
    return Y & np.uint64((1 << ell) - 1)


class Case:
    def __init__(self, nb, oracle, N, L, ell, L_out, m, n, kq, nq=1, impl=0, seed=0x5EED, W=None, X=None,
                 oracle_full=True, flags=0):
        self.nb, self.O = nb, oracle
        self.N, self.L, self.ell, self.L_out = N, L, ell, L_out
        self.m, self.n, self.kq, self.nq, self.k = m, n, kq, nq, kq * nq
        self.seed = seed
        self.ctx = nb.nimbus_ctx_create(N, L, ell, L_out, impl, flags=flags)
        self.pr = np.array(nb.nimbus_ctx_primes(self.ctx), np.uint32)
        self.W = ni.gen_W(seed, m, n, ell) if W is None else W
        self.X = ni.gen_X(seed ^ 0xA5, self.k, m, ell) if X is None else X
        self.sk = nb.nimbus_keygen(self.ctx, seed)
        self.encw = nb.nimbus_encrypt_weights(self.ctx, self.sk, dev_u32(self.W), seed)
        self.s_oracle = oracle.keygen(N, seed)
        self.E_oracle = oracle.encrypt_rows(N, L, self.pr, ell, self.s_oracle, self.W, seed) if oracle_full else None

    def run(self, mask_seed=None):
        nb = self.nb
        mask_seed = self.seed if mask_seed is None else mask_seed
        ws = nb.alloc_workspace(self.ctx, self.encw, self.k)
        cts, R = nb.alloc_outputs(self.ctx, self.encw, self.kq, self.nq)
        if os.environ.get("NIMBUS_TEST_HINT"):      # soak switch: every call carries a next-matmul prefetch hint
            nb.nimbus_cop_prefetch_next(self.ctx, self.encw)
        nb.nimbus_cop_matmul(self.ctx, self.encw, dev_u32(self.X), self.kq, self.nq, mask_seed, cts, R, ws)
        nb.nimbus_sync(self.ctx)
        return cts, R

    def oracle_out(self, mask_seed=None):
        mask_seed = self.seed if mask_seed is None else mask_seed
        return self.O.cop_matmul(self.N, self.L, self.L_out, self.pr, self.ell, self.E_oracle, self.X, self.n,
                                 self.kq, self.nq, mask_seed)

    def check_decrypt(self, cts, R):
        """Server step 5: Dec - mask = X.W mod t; invalid slots = -r."""
        nb = self.nb
        Z, M = nb.nimbus_decrypt(self.ctx, self.sk, cts, self.kq, self.nq, self.n, want_full=True)
        t = 1 << self.ell
        Y = matmul_mod_t(self.X, self.W, self.ell)
        Rn = u32(R).astype(np.uint64)
        assert (u32(Z).astype(np.uint64) == (Y + t - Rn) % t).all()
        Mn = u32(M)
        Rr = self.N // self.n
        nct = Mn.shape[0] // self.nq
        for tg in range(Mn.shape[0]):
            th = tg % nct
            rows = min(Rr, self.kq - th * Rr)
            mask = ni.uniform_mod_t(self.seed, 6, self.N, self.ell, start=tg * self.N).astype(np.uint64)
            inval = np.ones(self.N, bool)
            inval[: rows * self.n] = False
            assert (Mn[tg][inval] == (t - mask[inval]) % t).all()
        return Z


# ------------------------------------------------------------------ primitives
def test_prg_words(nb, oracle):
    for seed, dom, start in ((ni.seed_cfg(1), 1, 0), (ni.seed_cfg(4), 2, 12345), (7, 6, 1 << 33)):
        got = nb.nimbus_prg_words(seed, dom, start, 4096).cpu().numpy().view(np.uint64)
        assert (got == oracle.words(seed, dom, start, 4096)).all()


@pytest.mark.parametrize("N,L", [(64, 2), (4096, 2), (8192, 3)])
def test_keygen_and_primes(nb, oracle, N, L):
    ctx = nb.nimbus_ctx_create(N, L, 16, 1)
    assert nb.nimbus_ctx_primes(ctx) == [int(p) for p in oracle.primes(N, L)]
    sk = nb.nimbus_keygen(ctx, ni.seed_cfg(2) + N)
    s = nb.nimbus_sk_export(sk).cpu().numpy()
    assert (s == oracle.keygen(N, ni.seed_cfg(2) + N)).all()


@pytest.mark.parametrize("N,L", [(64, 2), (1024, 3), (4096, 2), (8192, 3)])
def test_ntt_negacyclic_product(nb, oracle, N, L):
    """K2 through the library's NTT vs the oracle's negacyclic product."""
    ctx = nb.nimbus_ctx_create(N, L, 16, 1)
    pr = nb.nimbus_ctx_primes(ctx)
    rng = np.random.default_rng(N)
    cnt = 2
    a = np.stack([np.stack([rng.integers(0, p, N, dtype=np.uint64) for p in pr]) for _ in range(cnt)]).astype(np.uint32)
    b = np.stack([np.stack([rng.integers(0, p, N, dtype=np.uint64) for p in pr]) for _ in range(cnt)]).astype(np.uint32)
    b[0, :, :] = 0
    b[0, :, 0] = 1          # identity
    c = u32(nb.nimbus_negacyclic_mul(ctx, dev_u32(a), dev_u32(b)))
    assert (c[0] == a[0]).all()
    for i in range(cnt):
        for l, p in enumerate(pr):
            want = oracle.negacyclic_schoolbook(N, p, a[i, l], b[i, l]) if N <= 64 else \
                oracle.negacyclic_ntt(N, p, a[i, l], b[i, l])
            assert (c[i, l] == want).all()


# ------------------------------------------------------------------ Enc(W)
@pytest.mark.parametrize("N,L,ell,m,n", [(64, 2, 16, 16, 20), (4096, 2, 16, 64, 64), (4096, 2, 16, 200, 4096),
                                         (8192, 3, 32, 130, 768)])
def test_encrypt_weights_parity(nb, oracle, N, L, ell, m, n):
    c = Case(nb, oracle, N, L, ell, 2 if ell == 32 else 1, m, n, kq=1)
    E = u32(nb.nimbus_encw_export(c.encw))
    assert E.shape == c.E_oracle.shape
    assert (E == c.E_oracle).all()
    # import(export) round trip reproduces the resident layout
    w2 = nb.nimbus_encw_import(c.ctx, dev_u32(E), n)
    assert (u32(nb.nimbus_encw_export(w2)) == E).all()


@pytest.mark.parametrize("N,L,ell,m,n", [(4096, 2, 16, 200, 700), (8192, 3, 32, 130, 768), (1024, 2, 8, 3, 5)])
def test_encrypt_weights_into(nb, oracle, N, L, ell, m, n):
    """Re-encryption into an existing handle (new weights and seed) equals a fresh
    encryption with that seed, bit for bit against the oracle; offloaded handles
    are refused."""
    c = Case(nb, oracle, N, L, ell, 2 if ell == 32 else 1, m, n, kq=1)
    W2 = ni.gen_W(c.seed + 9, m, n, ell)
    nb.nimbus_encrypt_weights_into(c.ctx, c.sk, dev_u32(W2), c.seed + 9, c.encw)
    E2 = oracle.encrypt_rows(N, L, c.pr, ell, c.s_oracle, W2, c.seed + 9)
    assert (u32(nb.nimbus_encw_export(c.encw)) == E2).all()
    nb.nimbus_encw_offload(c.encw)
    with pytest.raises(nb.NimbusError):
        nb.nimbus_encrypt_weights_into(c.ctx, c.sk, dev_u32(W2), 1, c.encw)


# ------------------------------------------------------------------ contraction (step 2)
@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("N,L,ell,k,m,n", [
    (64, 2, 16, 12, 16, 20),          # toy
    (4096, 2, 16, 16, 64, 64),        # C1
    (4096, 2, 16, 200, 300, 700),     # two M tiles, ragged k and m (3 k-blocks, last partial)
    (8192, 3, 32, 130, 200, 768),     # ell=32: 4 X slices, 7 accumulators, ragged
    (1024, 2, 8, 129, 257, 100),      # ell=8: 1 X slice
    (1024, 2, 16, 1, 1, 1),           # degenerate k = m = n = 1
])
def test_cop_accumulate_parity(nb, oracle, impl, N, L, ell, k, m, n):
    c = Case(nb, oracle, N, L, ell, 2 if ell == 32 else 1, m, n, kq=k, impl=impl)
    ws = nb.alloc_workspace(c.ctx, c.encw, k)
    Cg = u32(nb.nimbus_cop_accumulate(c.ctx, c.encw, dev_u32(c.X), ws))
    nb.nimbus_sync(c.ctx)
    Co = oracle.cop_accumulate(N, L, c.pr, c.E_oracle, c.X)
    assert (Cg == Co).all()


def test_cop_onehot_selects_row_ciphertext(nb, oracle):
    """x = e_beta gives c[alpha] = Enc(W_beta) bit for bit."""
    N, L, m = 4096, 2, 300
    X = np.zeros((160, m), np.uint32)
    for a in range(160):
        X[a, (a * 7) % m] = 1
    c = Case(nb, oracle, N, L, 16, 1, m, 500, kq=160, X=X, oracle_full=False)
    ws = nb.alloc_workspace(c.ctx, c.encw, 160)
    Cg = u32(nb.nimbus_cop_accumulate(c.ctx, c.encw, dev_u32(X), ws))
    E = u32(nb.nimbus_encw_export(c.encw))
    for a in range(160):
        assert (Cg[a] == E[(a * 7) % m]).all()


# ------------------------------------------------------------------ end to end (steps 2-4)
E2E = [
    # name, N, L, ell, L_out, m, n, kq, nq, impl
    ("toy_l16", 64, 2, 16, 1, 16, 20, 12, 1, 0),
    ("toy_l32", 64, 3, 32, 2, 16, 20, 12, 1, 0),
    ("C1", 4096, 2, 16, 1, 64, 64, 16, 1, 0),
    ("C1_cc", 4096, 2, 16, 1, 64, 64, 16, 1, 1),
    ("C2", 4096, 2, 16, 1, 768, 768, 128, 1, 0),
    ("C3", 4096, 2, 16, 1, 768, 3072, 128, 1, 0),
    ("C2_cc", 4096, 2, 16, 1, 768, 768, 128, 1, 1),
    ("multiquery_ragged", 4096, 2, 16, 1, 200, 700, 23, 3, 0),
    ("l32_multiquery", 8192, 3, 32, 2, 300, 768, 25, 2, 0),
    ("l32_to1limb", 8192, 3, 16, 1, 100, 1000, 17, 1, 0),
    ("n_equals_N", 1024, 2, 16, 1, 100, 1024, 5, 1, 0),
    ("n_half_plus_1", 1024, 2, 16, 1, 70, 513, 4, 1, 0),
    ("k_one", 4096, 2, 16, 1, 128, 64, 1, 1, 0),
    ("m_one", 4096, 2, 16, 1, 1, 64, 64, 1, 0),
    ("R_gt_k", 8192, 3, 32, 2, 64, 64, 7, 2, 0),
    # resident-X kernel with 3 and 4 limbs (4-wide pack items), and with fewer column tiles than SMs
    ("res_L3_v4", 8192, 3, 16, 1, 768, 1024, 128, 1, 0),
    ("res_L4_v4", 8192, 4, 16, 2, 200, 2048, 128, 1, 0),
    ("res_small_grid", 1024, 2, 16, 1, 130, 96, 100, 1, 0),
    # n = 1: R = N rows per packed ciphertext (the largest lazy sum in the pack)
    ("n_one", 1024, 2, 16, 1, 50, 1, 1031, 1, 0),
]


@pytest.mark.parametrize("case", E2E, ids=[c[0] for c in E2E])
def test_cop_matmul_parity(nb, oracle, case):
    name, N, L, ell, L_out, m, n, kq, nq, impl = case
    c = Case(nb, oracle, N, L, ell, L_out, m, n, kq, nq, impl, seed=ni.seed_mm(2, 0, len(name)))
    cts, R = c.run()
    cts_o, R_o = c.oracle_out()
    assert cts.shape == cts_o.shape
    assert (u32(cts) == cts_o).all(), "output ciphertexts differ"
    assert (u32(R) == R_o).all(), "client share R differs"
    c.check_decrypt(cts, R)


def test_host_buffer_api_matches_device(nb, oracle):
    c = Case(nb, oracle, 4096, 2, 16, 1, 768, 768, 128, oracle_full=False)
    cts_d, R_d = c.run()
    ws = nb.alloc_workspace(c.ctx, c.encw, c.k)
    cts_h, R_h = nb.alloc_outputs(c.ctx, c.encw, c.kq, c.nq, pin=True, device="cpu")
    Xh = torch.from_numpy(c.X.view(np.int32)).pin_memory()
    nb.nimbus_cop_matmul_host(c.ctx, c.encw, Xh, c.kq, c.nq, c.seed, cts_h, R_h, ws)
    assert torch.equal(cts_h, cts_d.cpu()) and torch.equal(R_h, R_d.cpu())
    # pageable host buffers (staged copies from / to pageable memory): same bytes, and mixed
    Xp = torch.from_numpy(c.X.view(np.int32).copy())
    cts_p, R_p = torch.zeros_like(cts_h, device="cpu"), torch.zeros_like(R_h, device="cpu")
    assert not Xp.is_pinned() and not cts_p.is_pinned()
    nb.nimbus_cop_matmul_host(c.ctx, c.encw, Xp, c.kq, c.nq, c.seed, cts_p, R_p, ws)
    assert torch.equal(cts_p, cts_h) and torch.equal(R_p, R_h)
    cts_h.zero_()
    nb.nimbus_cop_matmul_host(c.ctx, c.encw, Xp, c.kq, c.nq, c.seed, cts_h, R_p, ws)
    assert torch.equal(cts_h, cts_p)


def test_host_batch_matches_single_calls(nb, oracle):
    """nimbus_cop_matmul_host_batch (uploads / downloads pipelined over 8 staging
    slots) gives, for every job of a mixed list longer than the slot count, the
    bytes nimbus_cop_matmul gives for it; one job checked against the oracle; a
    job list with a device tensor or a bad shape is refused before any work."""
    N, L, ell, L_out = 4096, 2, 16, 1
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 21)
    shapes = [(128, 768, 768, 1), (64, 300, 700, 2), (128, 768, 3072, 1), (100, 1000, 500, 1), (16, 64, 64, 1),
              (128, 768, 768, 1), (33, 129, 5, 3)]
    encs = {}
    jobs, ref = [], []
    for i, (kq, m, n, nq) in enumerate(shapes):
        if (m, n) not in encs:
            W = ni.gen_W(140 + i, m, n, ell)
            encs[(m, n)] = (W, nb.nimbus_encrypt_weights(ctx, sk, dev_u32(W), 140 + i))
        W, w = encs[(m, n)]
        Xn = ni.gen_X(150 + i, kq * nq, m, ell)
        ws = nb.alloc_workspace(ctx, w, kq * nq)
        c0, R0 = nb.alloc_outputs(ctx, w, kq, nq)
        nb.nimbus_cop_matmul(ctx, w, dev_u32(Xn), kq, nq, 160 + i, c0, R0, ws)
        ref.append((c0.cpu(), R0.cpu()))
        cts, R = nb.alloc_outputs(ctx, w, kq, nq, pin=True, device="cpu")
        jobs.append(dict(encw=w, X=torch.from_numpy(Xn.view(np.int32)).pin_memory(), k_per_query=kq,
                         n_queries=nq, mask_seed=160 + i, cts=cts, R=R, Xn=Xn, W=W))
    nb.nimbus_sync(ctx)
    wsb = torch.empty(nb.nimbus_cop_workspace_size_host_batch(ctx, jobs), dtype=torch.uint8, device=DEV)
    nb.nimbus_cop_matmul_host_batch(ctx, jobs, wsb)
    for j, (c0, R0) in zip(jobs, ref):
        assert torch.equal(j["cts"], c0) and torch.equal(j["R"], R0)
    j = jobs[3]
    pr = np.array(nb.nimbus_ctx_primes(ctx), np.uint32)
    E = oracle.encrypt_rows(N, L, pr, ell, oracle.keygen(N, 21), j["W"], 143)
    cts_o, R_o = oracle.cop_matmul(N, L, L_out, pr, ell, E, j["Xn"], j["W"].shape[1], j["k_per_query"],
                                   j["n_queries"], j["mask_seed"])
    assert (u32(j["cts"]) == cts_o).all() and (u32(j["R"]) == R_o).all()
    # refused before any work: a device tensor, a workspace too small
    bad = dict(jobs[0], X=jobs[0]["X"].cuda())
    with pytest.raises(ValueError):
        nb.nimbus_cop_matmul_host_batch(ctx, [jobs[1], bad], wsb)
    with pytest.raises(nb.NimbusError):
        nb.nimbus_cop_matmul_host_batch(ctx, jobs, wsb[:1024])


def test_host_batch_same_x_groups(nb, oracle):
    """Host-buffer job list with same-X groups (Q, K, V of a layer share one pinned X):
    the group is uploaded once and runs as one resident-X launch; over several layers (groups of 3
    next to groups of 3 and single jobs, more jobs than staging slots) every job's ciphertexts and R
    equal the single device calls; one job checked against the oracle."""
    N, L, ell, L_out = 4096, 2, 16, 1
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 31)
    kq, m, n = 128, 768, 768
    Ws = [ni.gen_W(170 + i, m, n, ell) for i in range(4)]
    ws_ = [nb.nimbus_encrypt_weights(ctx, sk, dev_u32(W), 170 + i) for i, W in enumerate(Ws)]
    jobs, ref = [], []
    for layer in range(4):
        Xq = ni.gen_X(180 + layer, kq, m, ell)
        Xo = ni.gen_X(190 + layer, kq, m, ell)
        hq = torch.from_numpy(Xq.view(np.int32)).pin_memory()
        ho = torch.from_numpy(Xo.view(np.int32)).pin_memory()
        for p in range(4):                       # Q, K, V share hq; O has its own input
            Xn, hx = (Xq, hq) if p < 3 else (Xo, ho)
            seed = 200 + 4 * layer + p
            wsd = nb.alloc_workspace(ctx, ws_[p], kq)
            c0, R0 = nb.alloc_outputs(ctx, ws_[p], kq, 1)
            nb.nimbus_cop_matmul(ctx, ws_[p], dev_u32(Xn), kq, 1, seed, c0, R0, wsd)
            ref.append((c0.cpu(), R0.cpu()))
            cts, R = nb.alloc_outputs(ctx, ws_[p], kq, 1, pin=True, device="cpu")
            jobs.append(dict(encw=ws_[p], X=hx, k_per_query=kq, n_queries=1, mask_seed=seed, cts=cts, R=R,
                             Xn=Xn, p=p))
    nb.nimbus_sync(ctx)
    wsb = torch.empty(nb.nimbus_cop_workspace_size_host_batch(ctx, jobs), dtype=torch.uint8, device=DEV)
    for _ in range(2):
        for j in jobs:
            j["cts"].fill_(-1)
            j["R"].fill_(-1)
        nb.nimbus_cop_matmul_host_batch(ctx, jobs, wsb)
        for i, (j, (c0, R0)) in enumerate(zip(jobs, ref)):
            assert torch.equal(j["cts"], c0) and torch.equal(j["R"], R0), f"job {i}"
    j = jobs[5]                                   # layer 1, K
    pr = np.array(nb.nimbus_ctx_primes(ctx), np.uint32)
    E = oracle.encrypt_rows(N, L, pr, ell, oracle.keygen(N, 31), Ws[1], 171)
    cts_o, R_o = oracle.cop_matmul(N, L, L_out, pr, ell, E, j["Xn"], n, kq, 1, j["mask_seed"])
    assert (u32(j["cts"]) == cts_o).all() and (u32(j["R"]) == R_o).all()


def test_host_batch_u64(nb, oracle):
    """The same pipelined host-buffer list at ell = 64 (uint64 X / R)."""
    N, L, ell, L_out = 256, 5, 64, 3
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 9)
    shapes = [(33, 130, 100, 2), (7, 300, 128, 1), (64, 64, 256, 1), (20, 50, 60, 1)]
    jobs, ref = [], []
    for i, (kq, m, n, nq) in enumerate(shapes):
        w = nb.nimbus_encrypt_weights_u64(ctx, sk, _dev_u64(ni.gen_W(70 + i, m, n, ell)), 70 + i)
        X = _dev_u64(ni.gen_X(80 + i, kq * nq, m, ell))
        ws = nb.alloc_workspace(ctx, w, kq * nq)
        c0, R0 = nb.alloc_outputs_u64(ctx, w, kq, nq)
        nb.nimbus_cop_matmul_u64(ctx, w, X, kq, nq, 90 + i, c0, R0, ws)
        ref.append((c0.cpu(), R0.cpu()))
        jobs.append(dict(encw=w, X=X.cpu().pin_memory(), k_per_query=kq, n_queries=nq, mask_seed=90 + i,
                         cts=torch.zeros_like(c0, device="cpu").pin_memory(),
                         R=torch.zeros_like(R0, device="cpu").pin_memory()))
    nb.nimbus_sync(ctx)
    wsb = torch.empty(nb.nimbus_cop_workspace_size_host_batch(ctx, jobs, wide=True), dtype=torch.uint8, device=DEV)
    nb.nimbus_cop_matmul_host_batch(ctx, jobs, wsb, wide=True)
    for j, (c0, R0) in zip(jobs, ref):
        assert torch.equal(j["cts"], c0) and torch.equal(j["R"], R0)


# ------------------------------------------------------------------ full-size configs (sampled)
def _sampled_check(c, cts, n_samples=600, rng_seed=0):
    nct = cts.shape[1]
    rng = np.random.default_rng(rng_seed)
    sq = rng.integers(0, c.nq, n_samples).astype(np.uint32)
    st = rng.integers(0, nct, n_samples).astype(np.uint32)
    sJ = rng.integers(0, c.N, n_samples).astype(np.uint32)
    sJ[:8] = [0, 1, c.n - 1, c.n, c.N - 1, c.N - c.n, (c.N // c.n) * c.n - 1, c.N // 2]
    want = c.O.cop_matmul_sampled(c.N, c.L, c.L_out, c.pr, c.ell, c.E_oracle, c.X, c.n, c.kq, c.nq, c.seed,
                                  sq, st, sJ)
    g = u32(cts)
    got = np.stack([g[sq[i], st[i], :, :, sJ[i]] for i in range(n_samples)])
    assert (got == want).all()


@pytest.mark.parametrize("ell,L_out", [(32, 2), (16, 1)])
def test_c4_full_size(nb, oracle, ell, L_out):
    """C4: X 128x3072, W 3072x768, N=8192, 3 limbs (BASELINE.json configs[3]) at the
    launch configuration bench.py times; Enc(W) compared in full, outputs sampled,
    every slot checked through decryption."""
    cfg = ni.CONFIGS[4]
    lay = cfg.layers[0][2]
    seed = ni.seed_mm(4)
    c = Case(nb, oracle, cfg.N, cfg.L, ell, L_out, lay.m, lay.n, lay.k_per_query, seed=seed,
             W=ni.gen_W(seed, lay.m, lay.n, ell), X=ni.gen_X(seed, lay.k, lay.m, ell))
    assert (u32(nb.nimbus_encw_export(c.encw)) == c.E_oracle).all()
    cts, R = c.run()
    _sampled_check(c, cts)
    c.check_decrypt(cts, R)


@pytest.mark.parametrize("ell,proj", [(32, 0), (32, 4), (32, 5), (16, 0), (16, 4), (16, 5)])
def test_c5_layer_matmuls(nb, oracle, ell, proj):
    """C5: seq 512 x 4 queries (k=2048) on the Q (768x768), FFN-up (768x3072) and
    FFN-down (3072x768) shapes of layer 0, same launch as bench --config 5 (ell = 32: the
    packed contraction at S_x = 4) and --config 5l16 (ell = 16: S_x = 2)."""
    cfg = ni.CONFIGS[5] if ell == 32 else ni.CONFIGS_L16[5]
    li, pj, lay = cfg.layers[proj]
    seed = ni.seed_mm(5, li, pj)
    c = Case(nb, oracle, cfg.N, cfg.L, cfg.ell, cfg.L_out, lay.m, lay.n, lay.k_per_query, lay.n_queries,
             seed=seed, W=ni.gen_W(seed, lay.m, lay.n, cfg.ell), X=ni.gen_X(seed, lay.k, lay.m, cfg.ell),
             flags=nb.FLAG_LARGE_K)                      # bench --config 5 sets the k >= 512 layout hint
    assert (u32(nb.nimbus_encw_export(c.encw)) == c.E_oracle).all()
    cts, R = c.run()
    _sampled_check(c, cts, n_samples=300)
    c.check_decrypt(cts, R)


@pytest.mark.parametrize("n,n_next", [(768, 768), (768, 3000), (3000, 768), (3000, 3000), (768, 100)])
def test_prefetch_next_hint_parity(nb, oracle, n, n_next):
    """nimbus_cop_prefetch_next (the next matmul's Enc(W), whose first tiles the resident-X
    contraction prefetches towards L2) never changes a byte: plain and fused R = 1 kernels, the
    hinted Enc(W) mapped either way, a hint left pending and one whose Enc(W) is destroyed."""
    c = Case(nb, oracle, 4096, 2, 16, 1, 300, n, 100, seed=0x9F00 + n)
    W2 = ni.gen_W(77, 300, n_next, 16)
    nxt = nb.nimbus_encrypt_weights(c.ctx, c.sk, dev_u32(W2), 77)
    cts_o, R_o = c.oracle_out()
    for hint in (nxt, c.encw, None):
        nb.nimbus_cop_prefetch_next(c.ctx, hint)
        cts, R = c.run()
        assert "k_cop_tc_res" in nb.nimbus_last_contraction(c.ctx)
        assert (u32(cts) == cts_o).all() and (u32(R) == R_o).all()
    c.check_decrypt(cts, R)
    nb.nimbus_cop_prefetch_next(c.ctx, nxt)     # pending hint, its Enc(W) destroyed before the launch
    del nxt
    cts, R = c.run()
    assert (u32(cts) == cts_o).all() and (u32(R) == R_o).all()
    other = Case(nb, oracle, 4096, 2, 16, 1, 64, 64, 4, seed=5, oracle_full=False)
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_cop_prefetch_next(c.ctx, other.encw)       # an Enc(W) of another context
    assert e.value.status == -1


# ------------------------------------------------------------------ packed contraction (cop_pk.cu)
PACKED_CASES = [
    # N, L, ell, L_out, m, n, kq, nq            R = N/n; theta = nq * ceil(kq/R)
    (1024, 3, 32, 2, 200, 128, 300, 2),        # R = 8, 76 theta: two theta tiles of 48 (last ragged), ragged m
    (2048, 3, 32, 2, 600, 256, 190, 3),        # R = 8, 72 theta over 3 queries (tiles cross queries)
    (2048, 3, 32, 2, 600, 128, 100, 8),        # R = 16: 4 k-blocks per accumulator drain, KB = 5 -> 2 chunks
    (1024, 4, 32, 2, 300, 384, 100, 1),        # two dropped limbs (L - L_out = 2), R = 2
    (1024, 3, 32, 2, 129, 1024, 60, 1),        # n = N: R = 1, no wrapped term at all
    (1024, 3, 32, 2, 200, 128, 416, 2),        # 104 theta = 2 tiles of RT = 52 (4-row accumulator tail chunk)
    (8192, 3, 32, 2, 257, 768, 500, 1),        # C5 geometry (R = 10, 50 theta, the last one holding 0 of 10 rows... ragged)
    # ell <= 16: S_x = 2 (5 accumulators, theta tiles of RT = 64 or 72)
    (1024, 3, 16, 1, 200, 128, 300, 2),        # R = 8, 76 theta: RT = 64, two tiles (last ragged), ragged m
    (2048, 3, 16, 1, 600, 256, 190, 3),        # R = 8, 72 theta = one RT = 72 tile over 3 queries
    (2048, 3, 16, 1, 600, 128, 100, 8),        # R = 16: 4 k-blocks per accumulator drain, KB = 5 -> 2 chunks
    (1024, 3, 16, 1, 300, 384, 100, 1),        # two dropped limbs, R = 2
    (1024, 2, 16, 1, 129, 1024, 60, 1),        # n = N: R = 1, one dropped limb
    (2048, 3, 12, 1, 300, 128, 100, 8),        # ell = 12 (t = 2^12, complement over 16 bits)
    (8192, 3, 16, 1, 257, 768, 500, 1),        # C5@l16 geometry
]


@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,nq", PACKED_CASES)
def test_packed_parity(nb, oracle, monkeypatch, N, L, ell, L_out, m, n, kq, nq):
    """The packed contraction (the GEMM over K = (shift r, beta) that writes the packed,
    mod-switched, masked ciphertexts directly; the wrapped terms through the bitwise
    complement of x and the ColSum correction) is bit-exact vs the oracle, takes 2
    launches (slice + contraction), and equals the unpacked two-pass path."""
    c = Case(nb, oracle, N, L, ell, L_out, m, n, kq, nq, seed=7000 + N + m + n, flags=nb.FLAG_LARGE_K)
    before = nb.nimbus_launch_count(c.ctx)
    cts, R = c.run()
    import os
    if not os.environ.get("NIMBUS_NO_PACKED"):                # switch soaks run the unpacked path here
        assert nb.nimbus_launch_count(c.ctx) - before == 2, "packed path not taken"
        pair = ell > 16 and (n // 128) % 2 == 0 and (N // 128) % 2 == 0 and os.environ.get("NIMBUS_PK_PAIR") == "1"
        if not os.environ.get("NIMBUS_PK_CL"):
            assert ("P2" in nb.nimbus_last_contraction(c.ctx)) == pair, nb.nimbus_last_contraction(c.ctx)
    cts_o, R_o = c.oracle_out()
    assert (u32(cts) == cts_o).all(), "output ciphertexts differ"
    assert (u32(R) == R_o).all(), "client share R differs"
    c.check_decrypt(cts, R)
    monkeypatch.setenv("NIMBUS_NO_PACKED", "1")
    c2 = Case(nb, oracle, N, L, ell, L_out, m, n, kq, nq, seed=7000 + N + m + n, flags=nb.FLAG_LARGE_K,
              oracle_full=False)
    before = nb.nimbus_launch_count(c2.ctx)
    cts2, R2 = c2.run()
    assert nb.nimbus_launch_count(c2.ctx) - before == 3
    assert torch.equal(cts, cts2) and torch.equal(R, R2)


@pytest.mark.parametrize("order,epol", [("0", "0"), ("1", "1"), ("1", "2")])
@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,nq", [PACKED_CASES[i] for i in (1, 3, 4, 6, 9, 13)])
def test_packed_unit_order_parity(nb, oracle, monkeypatch, order, epol, N, L, ell, L_out, m, n, kq, nq):
    """The packed contraction's unit order (NIMBUS_PK_ORDER: 1 = theta groups fastest and the J tiles
    walked in shift order, the default; 0 = J tiles fastest) and the L2 policy of its Enc(W) copies
    (NIMBUS_PK_EPOL) change which CTA computes which tile and when, never a byte of the output."""
    monkeypatch.setenv("NIMBUS_PK_ORDER", order)
    monkeypatch.setenv("NIMBUS_PK_EPOL", epol)
    c = Case(nb, oracle, N, L, ell, L_out, m, n, kq, nq, seed=7200 + N + m + n, flags=nb.FLAG_LARGE_K)
    cts, R = c.run()
    cts_o, R_o = c.oracle_out()
    assert (u32(cts) == cts_o).all() and (u32(R) == R_o).all()
    c.check_decrypt(cts, R)


@pytest.mark.parametrize("rt", ["48", "52", "56", "64"])
@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,nq", [c for c in PACKED_CASES if c[2] > 16 and (c[5] // 128) % 2 == 0])
def test_packed_pair_parity(nb, oracle, monkeypatch, rt, N, L, ell, L_out, m, n, kq, nq):
    """The opt-in CTA-pair form of the packed contraction (NIMBUS_PK_PAIR=1: tcgen05 cta_group::2,
    M = 256 over two J tiles, the X block split between the pair) is bit-exact vs the oracle, at
    every theta-tile height (N = S_x RT = 192 / 208 / 224 / 256)."""
    monkeypatch.setenv("NIMBUS_PK_PAIR", "1")
    monkeypatch.setenv("NIMBUS_PK_RT", rt)
    c = Case(nb, oracle, N, L, ell, L_out, m, n, kq, nq, seed=7100 + N + m + n, flags=nb.FLAG_LARGE_K)
    cts, R = c.run()
    assert f"{rt}, 2, P2" in nb.nimbus_last_contraction(c.ctx)
    cts_o, R_o = c.oracle_out()
    assert (u32(cts) == cts_o).all() and (u32(R) == R_o).all()
    c.check_decrypt(cts, R)


@pytest.mark.parametrize("ell,L_out,pair", [(32, 2, 0), (16, 1, 0), (32, 2, 1)])
def test_packed_batch_parity(nb, oracle, monkeypatch, ell, L_out, pair):
    """A C5-like job list (Q/up/down shapes at a small N) as ONE packed slice launch
    and ONE packed contraction launch: every job bit-exact vs the oracle (S_x = 4 and 2,
    and the opt-in CTA-pair form)."""
    if pair:
        monkeypatch.setenv("NIMBUS_PK_PAIR", "1")
    N, L = 2048, 3
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out, flags=nb.FLAG_LARGE_K)
    pr = np.array(nb.nimbus_ctx_primes(ctx), np.uint32)
    sk = nb.nimbus_keygen(ctx, 77)
    s = oracle.keygen(N, 77)
    shapes = [(200, 256, 256, 2), (160, 256, 1024, 2), (200, 700, 256, 2), (130, 256, 256, 3)]   # >= 48 theta each
    jobs = []
    for i, (kq, m, n, nq) in enumerate(shapes):
        W = ni.gen_W(500 + i, m, n, ell)
        X = ni.gen_X(600 + i, kq * nq, m, ell)
        w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(W), 500 + i)
        cts, R = nb.alloc_outputs(ctx, w, kq, nq)
        jobs.append(dict(encw=w, X=dev_u32(X), k_per_query=kq, n_queries=nq, mask_seed=900 + i, cts=cts, R=R,
                         W=W, Xh=X))
    ws = torch.empty(nb.nimbus_cop_workspace_size_batch(ctx, jobs), dtype=torch.uint8, device=DEV)
    before = nb.nimbus_launch_count(ctx)
    nb.nimbus_cop_matmul_batch(ctx, jobs, ws)
    nb.nimbus_sync(ctx)
    import os
    if not os.environ.get("NIMBUS_NO_PACKED"):
        assert nb.nimbus_launch_count(ctx) - before == 2
    for i, j in enumerate(jobs):
        E = oracle.encrypt_rows(N, L, pr, ell, s, j["W"], 500 + i)
        cts_o, R_o = oracle.cop_matmul(N, L, L_out, pr, ell, E, j["Xh"], j["W"].shape[1], j["k_per_query"],
                                       j["n_queries"], j["mask_seed"])
        assert (u32(j["cts"]) == cts_o).all() and (u32(j["R"]) == R_o).all(), f"job {i}"


@pytest.mark.parametrize("N,m,n,kq", [(4096, 300, 700, 70), (1024, 100, 200, 128), (2048, 768, 300, 33),
                                      (256, 700, 100, 128)])
def test_same_x_group_batch_parity(nb, oracle, N, m, n, kq):
    """Q, K, V of a layer share their input X: in a batch, consecutive jobs with
    the same X and shape run as ONE slice + ONE resident-X contraction over their three Enc(W)s
    + ONE pack launch; the output ciphertexts and R of every job are bit-exact vs the oracle,
    and a following job with its own X (O) takes the per-job path.  Shapes: 1, 2 and 3 k-block
    pairs in the first tile, and fewer column tiles than SMs (N = 256)."""
    L, ell, L_out = 2, 16, 1
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    pr = np.array(nb.nimbus_ctx_primes(ctx), np.uint32)
    sk = nb.nimbus_keygen(ctx, 55)
    s = oracle.keygen(N, 55)
    nq = 1
    Xq = ni.gen_X(56, kq * nq, m, ell)
    Xo = ni.gen_X(57, kq * nq, m, ell)
    dXq, dXo = dev_u32(Xq), dev_u32(Xo)
    jobs = []
    for i in range(4):
        W = ni.gen_W(560 + i, m, n, ell)
        w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(W), 560 + i)
        cts, R = nb.alloc_outputs(ctx, w, kq, nq)
        jobs.append(dict(encw=w, X=dXq if i < 3 else dXo, k_per_query=kq, n_queries=nq, mask_seed=570 + i,
                         cts=cts, R=R, W=W, Xh=Xq if i < 3 else Xo))
    ws = torch.empty(nb.nimbus_cop_workspace_size_batch(ctx, jobs), dtype=torch.uint8, device=DEV)
    before = nb.nimbus_launch_count(ctx)
    nb.nimbus_cop_matmul_batch(ctx, jobs, ws)
    nb.nimbus_sync(ctx)
    import os
    if not (os.environ.get("NIMBUS_NO_GROUP") or os.environ.get("NIMBUS_RES", "1") != "1"):   # switch soaks
        assert nb.nimbus_launch_count(ctx) - before == 3 + 3, "group (3 launches) + O (3 launches)"
    for i, j in enumerate(jobs):
        E = oracle.encrypt_rows(N, L, pr, ell, s, j["W"], 560 + i)
        cts_o, R_o = oracle.cop_matmul(N, L, L_out, pr, ell, E, j["Xh"], n, kq, nq, j["mask_seed"])
        assert (u32(j["cts"]) == cts_o).all() and (u32(j["R"]) == R_o).all(), f"job {i}"


# ------------------------------------------------------------------ errors
def test_error_codes(nb, oracle):
    ctx = nb.nimbus_ctx_create(1024, 2, 16, 1)
    sk = nb.nimbus_keygen(ctx, 1)
    W = dev_u32(ni.gen_W(1, 4, 1025, 16))
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_encrypt_weights(ctx, sk, W, 1)     # n > N
    assert e.value.status == -2
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_ctx_create(1000, 2, 16, 1)          # N not a power of two
    assert e.value.status == -1
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_ctx_create(1024, 2, 16, 3)          # L_out > L
    assert e.value.status == -1
    # ell=32 cannot be switched down to one 31-bit limb: the noise bound refuses it
    ctx32 = nb.nimbus_ctx_create(8192, 3, 32, 1)
    sk32 = nb.nimbus_keygen(ctx32, 1)
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_encrypt_weights(ctx32, sk32, dev_u32(ni.gen_W(1, 8, 8, 32)), 1)
    assert e.value.status == -4
    # range check: an entry >= t is reported at the next sync
    ctxr = nb.nimbus_ctx_create(1024, 2, 16, 1, flags=nb.FLAG_CHECK_RANGE)
    skr = nb.nimbus_keygen(ctxr, 1)
    wr = nb.nimbus_encrypt_weights(ctxr, skr, dev_u32(ni.gen_W(1, 8, 8, 16)), 1)
    ws = nb.alloc_workspace(ctxr, wr, 4)
    cts, R = nb.alloc_outputs(ctxr, wr, 4, 1)
    Xbad = ni.gen_X(1, 4, 8, 16)
    Xbad[2, 3] = 1 << 16
    nb.nimbus_cop_matmul(ctxr, wr, dev_u32(Xbad), 4, 1, 1, cts, R, ws)
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_sync(ctxr)
    assert e.value.status == -3
    # workspace too small
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_cop_matmul(ctxr, wr, dev_u32(ni.gen_X(1, 4, 8, 16)), 4, 1, 1, cts, R, ws[:16])
    assert e.value.status == -2


def test_handles_outlive_context(nb, oracle):
    """Handles hold a reference to their context (nimbus_ctx_destroy): destroying the context
    first, then its handles in any order, leaves no CUDA error behind, and the next context's
    calls run clean (cyclic garbage collection frees Python handles in arbitrary order)."""
    for order in ("encw_first", "sk_first"):
        ctx = nb.nimbus_ctx_create(256, 2, 16, 1)
        sk = nb.nimbus_keygen(ctx, 1)
        pk = nb.nimbus_keygen_pk(ctx, sk, 2)
        w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(1, 8, 8, 16)), 1)
        ctx.close()
        for h in ((w, pk, sk) if order == "encw_first" else (sk, pk, w)):
            h.close()
    torch.cuda.synchronize()
    c = Case(nb, oracle, 256, 2, 16, 1, 40, 24, 9, 1, seed=77)
    cts, R = c.run()
    cts_o, R_o = c.oracle_out()
    assert (u32(cts) == cts_o).all() and (u32(R) == R_o).all()


@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,n2,flags", [
    (4096, 2, 16, 1, 300, 768, 128, 500, 0),      # pack (R = 5) -> resident-X slice
    (4096, 2, 16, 1, 300, 3072, 128, 700, 0),     # fused R = 1 contraction -> slice
    (1024, 3, 32, 2, 200, 128, 512, 256, 1),      # packed contraction (C5 path) -> packed slice
    (1024, 3, 16, 1, 200, 128, 512, 256, 1),      # the same at S_x = 2 (C5@l16 path)
])
def test_output_feeds_next_input(nb, oracle, N, L, ell, L_out, m, n, kq, n2, flags):
    """The client share R of one call used as X of the next call on the same stream, with no
    synchronisation in between: the slice kernels normally read X before their PDL wait, but
    X is an output of the kernel right before them (which triggers its dependents early), so
    they must read it after the wait (pdl_outputs_overlap).  Both calls bit-exact vs the oracle."""
    fl = nb.FLAG_LARGE_K if flags else 0
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out, flags=fl)
    pr = np.array(nb.nimbus_ctx_primes(ctx), np.uint32)
    sk = nb.nimbus_keygen(ctx, 91)
    s = oracle.keygen(N, 91)
    W1, W2 = ni.gen_W(92, m, n, ell), ni.gen_W(93, n, n2, ell)
    X1 = ni.gen_X(94, kq, m, ell)
    w1 = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(W1), 92)
    w2 = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(W2), 93)
    ws1, ws2 = nb.alloc_workspace(ctx, w1, kq), nb.alloc_workspace(ctx, w2, kq)
    c1, R1 = nb.alloc_outputs(ctx, w1, kq, 1)
    c2, R2 = nb.alloc_outputs(ctx, w2, kq, 1)
    nb.nimbus_sync(ctx)
    for _ in range(3):                   # a few times: the race, if any, is timing-dependent
        R1.fill_(-1)
        torch.cuda.synchronize()
        nb.nimbus_cop_matmul(ctx, w1, dev_u32(X1), kq, 1, 95, c1, R1, ws1)
        nb.nimbus_cop_matmul(ctx, w2, R1, kq, 1, 96, c2, R2, ws2)     # X of call 2 = R of call 1
        nb.nimbus_sync(ctx)
        E1 = oracle.encrypt_rows(N, L, pr, ell, s, W1, 92)
        cts_o, R_o = oracle.cop_matmul(N, L, L_out, pr, ell, E1, X1, n, kq, 1, 95)
        assert (u32(c1) == cts_o).all() and (u32(R1) == R_o).all()
        E2 = oracle.encrypt_rows(N, L, pr, ell, s, W2, 93)
        cts2_o, R2_o = oracle.cop_matmul(N, L, L_out, pr, ell, E2, R_o, n2, kq, 1, 96)
        assert (u32(c2) == cts2_o).all() and (u32(R2) == R2_o).all()


def test_batch_matches_sequential_and_oracle(nb, oracle):
    """nimbus_cop_matmul_batch (pack of job i overlapped with the contraction of
    job i+1 on a side stream) gives the same bytes as job-by-job calls, and the
    oracle's, for a mixed sequence of shapes sharing one context."""
    N, L, ell, L_out = 4096, 2, 16, 1
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    pr = np.array(nb.nimbus_ctx_primes(ctx), np.uint32)
    sk = nb.nimbus_keygen(ctx, 91)
    shapes = [(128, 768, 768, 1), (64, 300, 700, 2), (128, 768, 3072, 1), (100, 1000, 500, 1), (20, 64, 64, 3)]
    jobs, seq = [], []
    for i, (kq, m, n, nq) in enumerate(shapes):
        W = ni.gen_W(100 + i, m, n, ell)
        X = ni.gen_X(200 + i, kq * nq, m, ell)
        w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(W), 100 + i)
        cts, R = nb.alloc_outputs(ctx, w, kq, nq)
        jobs.append(dict(encw=w, X=dev_u32(X), k_per_query=kq, n_queries=nq, mask_seed=300 + i, cts=cts, R=R,
                         W=W, Xh=X))
    ws = torch.empty(nb.nimbus_cop_workspace_size_batch(ctx, jobs), dtype=torch.uint8, device=DEV)
    nb.nimbus_cop_matmul_batch(ctx, jobs, ws)
    nb.nimbus_sync(ctx)
    for j in jobs:
        kq, nq = j["k_per_query"], j["n_queries"]
        ws1 = nb.alloc_workspace(ctx, j["encw"], kq * nq)
        c2, R2 = nb.alloc_outputs(ctx, j["encw"], kq, nq)
        nb.nimbus_cop_matmul(ctx, j["encw"], j["X"], kq, nq, j["mask_seed"], c2, R2, ws1)
        nb.nimbus_sync(ctx)
        assert torch.equal(c2, j["cts"]) and torch.equal(R2, j["R"])
    j = jobs[1]
    s = oracle.keygen(N, 91)
    E = oracle.encrypt_rows(N, L, pr, ell, s, j["W"], 101)
    cts_o, R_o = oracle.cop_matmul(N, L, L_out, pr, ell, E, j["Xh"], j["W"].shape[1], j["k_per_query"],
                                   j["n_queries"], j["mask_seed"])
    assert (u32(j["cts"]) == cts_o).all() and (u32(j["R"]) == R_o).all()


@pytest.mark.parametrize("env", [{"NIMBUS_TRANSPOSED": "1"}, {"NIMBUS_TRANSPOSED": "1", "NIMBUS_T_RT": "32"},
                                 {"NIMBUS_NO_RESIDENT": "1"}, {"NIMBUS_CLUSTER": "2"},
                                 {"NIMBUS_NO_RESIDENT": "1", "NIMBUS_CLUSTER": "2"}, {"NIMBUS_RES": "1"},
                                 {"NIMBUS_RES": "2"}, {"NIMBUS_PACK_V": "1"}, {"NIMBUS_PACK_V": "2"},
                                 {"NIMBUS_PACK_V": "4"}])
@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,nq", [(4096, 2, 16, 1, 768, 768, 128, 1),
                                                     (8192, 3, 32, 2, 300, 1000, 70, 3)])
def test_kernel_variants_parity(nb, oracle, monkeypatch, env, N, L, ell, L_out, m, n, kq, nq):
    """The non-default kernel variants (transposed kernel for ell=32, 48-column
    streaming kernel for ell=16, 2-CTA clusters with X multicast) give the same
    bytes as the oracle."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    c = Case(nb, oracle, N, L, ell, L_out, m, n, kq, nq, seed=777 + m)
    cts, R = c.run()
    cts_o, R_o = c.oracle_out()
    assert (u32(cts) == cts_o).all() and (u32(R) == R_o).all()


@pytest.mark.parametrize("res", ["1", "2"])
@pytest.mark.parametrize("m,n,kq,nq", [(64, 64, 16, 1), (129, 200, 128, 1), (300, 1000, 70, 1), (520, 768, 33, 2),
                                       (640, 3072, 128, 1), (768, 5, 128, 1)])
def test_resident_kernels_parity(nb, oracle, monkeypatch, res, m, n, kq, nq):
    """Both resident-X contraction kernels (ell = 16, k <= 128, m <= 768): k-block
    counts 1..6 (odd counts leave a half k-block pair; from k-block 4 on slice 1
    sits in shared memory in the deep-ring kernel), ragged rows and columns."""
    monkeypatch.setenv("NIMBUS_RES", res)
    c = Case(nb, oracle, 4096, 2, 16, 1, m, n, kq, nq, seed=4242 + m + n)
    cts, R = c.run()
    cts_o, R_o = c.oracle_out()
    assert (u32(cts) == cts_o).all() and (u32(R) == R_o).all()


@pytest.mark.parametrize("fuse", ["1", "0"])
@pytest.mark.parametrize("N,m,n,kq,nq", [(4096, 768, 3072, 128, 1), (4096, 129, 2049, 100, 1),
                                         (4096, 520, 4096, 33, 2), (256, 64, 129, 128, 1), (64, 300, 37, 17, 3)])
def test_fused_r1_parity(nb, oracle, monkeypatch, fuse, N, m, n, kq, nq):
    """R = 1 layers (n > N/2, L = 2 -> L_out = 1, ell = 16, k <= 128): the resident
    contraction's epilogue does the mod-switch and the mask and writes the output
    ciphertexts and R itself (2 launches: slice + contraction; NIMBUS_NO_FUSE=1 keeps
    the separate pack, 3 launches).  Both are bit-exact vs the oracle: C3, ragged
    n (R tail not a multiple of 8), ragged rows and k-blocks, n = N with two
    queries, and grids smaller than the SM count (N = 256, 64)."""
    monkeypatch.setenv("NIMBUS_NO_FUSE", "0" if fuse == "1" else "1")
    c = Case(nb, oracle, N, 2, 16, 1, m, n, kq, nq, seed=9090 + m + n)
    before = nb.nimbus_launch_count(c.ctx)
    cts, R = c.run()
    assert nb.nimbus_launch_count(c.ctx) - before == (2 if fuse == "1" else 3)
    cts_o, R_o = c.oracle_out()
    assert (u32(cts) == cts_o).all(), "output ciphertexts differ"
    assert (u32(R) == R_o).all(), "client share R differs"
    c.check_decrypt(cts, R)
    # host-buffer call (R produced by its own kernel, the fused epilogue skips it): same bytes
    ws = nb.alloc_workspace(c.ctx, c.encw, c.k)
    cts_h, R_h = nb.alloc_outputs(c.ctx, c.encw, c.kq, c.nq, pin=True, device="cpu")
    Xh = torch.from_numpy(c.X.view(np.int32)).pin_memory()
    nb.nimbus_cop_matmul_host(c.ctx, c.encw, Xh, c.kq, c.nq, c.seed, cts_h, R_h, ws)
    assert torch.equal(cts_h, cts.cpu()) and torch.equal(R_h, R.cpu())


# ------------------------------------------------------------------ server, Alg. 1 step 5
@pytest.mark.parametrize("ell", [8, 12, 16, 32])
@pytest.mark.parametrize("k,m,n", [(1, 1, 1), (200, 300, 100), (128, 768, 768), (130, 129, 65)])
def test_plain_matmul_parity(nb, oracle, ell, k, m, n):
    """nimbus_plain_matmul (int8-sliced tcgen05 GEMM mod 2^ell) == oracle.plain_matmul,
    bit for bit, with and without the added term; ragged k, m, n tails."""
    N = 4096 if ell <= 16 else 8192
    ctx = nb.nimbus_ctx_create(N, 2 if ell <= 16 else 3, ell, 1 if ell <= 16 else 2)
    W = ni.gen_W(11 + m, m, n, ell)
    X = ni.gen_X(12 + k, k, m, ell)
    w = nb.nimbus_plain_weights(ctx, dev_u32(W))
    Y = nb.nimbus_plain_matmul(ctx, w, dev_u32(X))
    want = oracle.plain_matmul(X, W, ell)
    assert (u32(Y) == want).all()
    A = ni.gen_X(13, k, n, ell)
    Y2 = nb.nimbus_plain_matmul(ctx, w, dev_u32(X), add=dev_u32(A))
    t = np.uint64((1 << ell) - 1)
    assert (u32(Y2) == ((want.astype(np.uint64) + A) & t)).all()


@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,nq", [(4096, 2, 16, 1, 768, 768, 128, 1),
                                                     (4096, 2, 16, 1, 200, 700, 23, 3),
                                                     (8192, 3, 32, 2, 300, 768, 25, 2),
                                                     (4096, 2, 16, 1, 768, 3072, 128, 1)])
def test_server_output_parity_and_shares(nb, oracle, N, L, ell, L_out, m, n, kq, nq):
    """Alg. 1 end to end on the GPU: client COP (nimbus_cop_matmul) + server step 5
    (nimbus_server_output).  <Y>_s equals the oracle's bit for bit, and
    <Y>_s + <Y>_c (= R) reconstructs X.W mod t for X = <X>_s + <X>_c."""
    c = Case(nb, oracle, N, L, ell, L_out, m, n, kq, nq, seed=4242 + m, oracle_full=False)
    cts, R = c.run()
    Xs = ni.gen_X(c.seed + 7, c.k, m, ell)
    w = nb.nimbus_plain_weights(c.ctx, dev_u32(c.W))
    Ys = nb.nimbus_server_output(c.ctx, c.sk, w, dev_u32(Xs), cts, kq, nq)
    nb.nimbus_sync(c.ctx)
    want = oracle.server_output(N, L_out, c.pr[:L_out], ell, c.s_oracle, u32(cts), Xs, c.W, kq, nq)
    assert (u32(Ys) == want).all()
    t = (1 << ell)
    X = (c.X.astype(np.uint64) + Xs) % t
    Y = matmul_mod_t(X, c.W, ell)
    assert ((u32(Ys).astype(np.uint64) + u32(R)) % t == Y).all()


# ------------------------------------------------------------------ streamed Enc(W) (host-resident)
def _oracle_job(oracle, N, L, L_out, ell, sk_seed, w_seed, x_seed, shape, mask_seed):
    """The oracle's (cts, R) for one job of the streamed-path tests (W, X from their seeds)."""
    kq, m, n, nq = shape
    pr = oracle.primes(N, L)
    s = oracle.keygen(N, sk_seed)
    W = ni.gen_W(w_seed, m, n, ell)
    E = oracle.encrypt_rows(N, L, pr, ell, s, W, w_seed)
    return oracle.cop_matmul(N, L, L_out, pr, ell, E, ni.gen_X(x_seed, kq * nq, m, ell), n, kq, nq, mask_seed)


def test_streamed_matches_resident(nb, oracle):
    """nimbus_cop_matmul_streamed (Enc(W) offloaded to pinned host memory and
    staged into alternating device slots, copy j+2 overlapping compute j+1) gives
    the bytes nimbus_cop_matmul gives with Enc(W) resident, for a job list mixing
    host-resident and resident matrices of different shapes; offloaded handles
    are refused by nimbus_cop_matmul and work again after nimbus_encw_reload."""
    N, L, ell, L_out = 4096, 2, 16, 1
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 5)
    shapes = [(128, 768, 768, 1), (64, 300, 700, 2), (128, 768, 3072, 1), (100, 1000, 500, 1), (128, 768, 768, 1)]
    jobs, ref = [], []
    ws = torch.empty(max(nb.nimbus_cop_workspace_size(ctx, nb.nimbus_encrypt_weights(ctx, sk, dev_u32(
        ni.gen_W(1, m, n, ell)), 1), kq * nq) for kq, m, n, nq in shapes), dtype=torch.uint8, device=DEV)
    for i, (kq, m, n, nq) in enumerate(shapes):
        w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(40 + i, m, n, ell)), 40 + i)
        X = dev_u32(ni.gen_X(50 + i, kq * nq, m, ell))
        c0, R0 = nb.alloc_outputs(ctx, w, kq, nq)
        nb.nimbus_cop_matmul(ctx, w, X, kq, nq, 60 + i, c0, R0, ws)
        ref.append((c0, R0))
        cts, R = nb.alloc_outputs(ctx, w, kq, nq)
        jobs.append(dict(encw=w, X=X, k_per_query=kq, n_queries=nq, mask_seed=60 + i, cts=cts, R=R))
    nb.nimbus_sync(ctx)
    for i in (0, 2, 3, 4):                      # job 1 stays resident
        nb.nimbus_encw_offload(jobs[i]["encw"])
        assert not nb.nimbus_encw_is_resident(jobs[i]["encw"])
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_cop_matmul(ctx, jobs[0]["encw"], jobs[0]["X"], 128, 1, 60, jobs[0]["cts"], jobs[0]["R"], ws)
    assert e.value.status == -1
    stage = torch.empty(nb.nimbus_cop_stage_size(ctx, jobs), dtype=torch.uint8, device=DEV)
    nb.nimbus_cop_matmul_streamed(ctx, jobs, ws, stage)
    nb.nimbus_sync(ctx)
    for i, (j, (c0, R0)) in enumerate(zip(jobs, ref)):
        assert torch.equal(j["cts"], c0) and torch.equal(j["R"], R0)
        # and the oracle's bytes, independently of the resident path
        cts_o, R_o = _oracle_job(oracle, N, L, L_out, ell, 5, 40 + i, 50 + i, shapes[i], 60 + i)
        assert (u32(j["cts"]) == cts_o).all() and (u32(j["R"]) == R_o).all(), f"job {i}"
    nb.nimbus_encw_reload(jobs[0]["encw"])
    c1, R1 = nb.alloc_outputs(ctx, jobs[0]["encw"], 128, 1)
    nb.nimbus_cop_matmul(ctx, jobs[0]["encw"], jobs[0]["X"], 128, 1, 60, c1, R1, ws)
    nb.nimbus_sync(ctx)
    assert torch.equal(c1, ref[0][0]) and torch.equal(R1, ref[0][1])


def test_streamed_from_files(nb, oracle, tmp_path):
    """Enc(W) kept on disk: store files opened as file-backed
    handles are read, uploaded and tiled per job by nimbus_cop_matmul_streamed; a job
    list mixing resident, host-offloaded and file-backed matrices (more file jobs than
    read buffers) gives the bytes of resident calls.  Opening a truncated or corrupt
    file fails with NIMBUS_EIO (the corrupt one only with verify); a file that vanishes
    after opening makes nimbus_sync report NIMBUS_EIO; nimbus_encw_reload reads a
    file-backed handle into HBM."""
    N, L, ell, L_out = 4096, 2, 16, 1
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 6)
    shapes = [(128, 768, 768, 1), (64, 300, 700, 2), (128, 768, 3072, 1), (100, 1000, 500, 1), (33, 129, 64, 1),
              (128, 768, 768, 1)]
    kinds = ["file", "resident", "file", "host", "file", "file"]
    jobs, ref, paths = [], [], []
    ws = torch.empty(max(nb.nimbus_cop_workspace_size(ctx, nb.nimbus_encrypt_weights(ctx, sk, dev_u32(
        ni.gen_W(1, m, n, ell)), 1), kq * nq) for kq, m, n, nq in shapes), dtype=torch.uint8, device=DEV)
    for i, ((kq, m, n, nq), kind) in enumerate(zip(shapes, kinds)):
        w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(40 + i, m, n, ell)), 40 + i)
        X = dev_u32(ni.gen_X(50 + i, kq * nq, m, ell))
        c0, R0 = nb.alloc_outputs(ctx, w, kq, nq)
        nb.nimbus_cop_matmul(ctx, w, X, kq, nq, 60 + i, c0, R0, ws)
        ref.append((c0, R0))
        if kind == "file":
            path = str(tmp_path / f"w{i}.nimbus")
            nb.nimbus_encw_save(w, path)
            paths.append(path)
            w = nb.nimbus_encw_open(ctx, path, verify=(i == 0))
            assert not nb.nimbus_encw_is_resident(w)
        elif kind == "host":
            nb.nimbus_encw_offload(w)
        cts, R = nb.alloc_outputs(ctx, w, kq, nq)
        jobs.append(dict(encw=w, X=X, k_per_query=kq, n_queries=nq, mask_seed=60 + i, cts=cts, R=R))
    nb.nimbus_sync(ctx)
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_cop_matmul(ctx, jobs[0]["encw"], jobs[0]["X"], 128, 1, 60, jobs[0]["cts"], jobs[0]["R"], ws)
    assert e.value.status == -1
    stage = torch.empty(nb.nimbus_cop_stage_size(ctx, jobs), dtype=torch.uint8, device=DEV)
    for rep in range(2):
        for j in jobs:
            j["cts"].zero_()
            j["R"].zero_()
        nb.nimbus_cop_matmul_streamed(ctx, jobs, ws, stage)
        nb.nimbus_sync(ctx)
        for i, (j, (c0, R0)) in enumerate(zip(jobs, ref)):
            assert torch.equal(j["cts"], c0) and torch.equal(j["R"], R0)
            if rep == 0:      # the oracle's bytes, independently of the resident path
                cts_o, R_o = _oracle_job(oracle, N, L, L_out, ell, 6, 40 + i, 50 + i, shapes[i], 60 + i)
                assert (u32(j["cts"]) == cts_o).all() and (u32(j["R"]) == R_o).all(), f"job {i} ({kinds[i]})"
    # reload a file-backed handle into HBM: plain calls work again
    nb.nimbus_encw_reload(jobs[0]["encw"])
    c1, R1 = nb.alloc_outputs(ctx, jobs[0]["encw"], 128, 1)
    nb.nimbus_cop_matmul(ctx, jobs[0]["encw"], jobs[0]["X"], 128, 1, 60, c1, R1, ws)
    nb.nimbus_sync(ctx)
    assert torch.equal(c1, ref[0][0]) and torch.equal(R1, ref[0][1])
    # truncated / corrupt files
    data = open(paths[1], "rb").read()
    trunc = str(tmp_path / "trunc.nimbus")
    open(trunc, "wb").write(data[:-100])
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_encw_open(ctx, trunc)
    assert e.value.status == -7
    bad = bytearray(data)
    bad[len(bad) // 2] ^= 0x40
    corrupt = str(tmp_path / "corrupt.nimbus")
    open(corrupt, "wb").write(bytes(bad))
    nb.nimbus_encw_open(ctx, corrupt)                      # header and size are fine
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_encw_open(ctx, corrupt, verify=True)
    assert e.value.status == -7
    # a file removed after opening: the streamed call's read fails, nimbus_sync reports it
    gone = str(tmp_path / "gone.nimbus")
    open(gone, "wb").write(data)
    wg = nb.nimbus_encw_open(ctx, gone)
    import os
    os.remove(gone)
    jg = dict(jobs[2], encw=wg)
    stage2 = torch.empty(nb.nimbus_cop_stage_size(ctx, [jg]), dtype=torch.uint8, device=DEV)
    nb.nimbus_cop_matmul_streamed(ctx, [jg], ws, stage2)
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_sync(ctx)
    assert e.value.status == -7


# ------------------------------------------------------------------ ell = 64 (the paper's t, 5 limbs)
def _u64(t):
    from paper_2411_15707_b200 import nimbus
    return nimbus.to_numpy_u64(t)


def _dev_u64(a):
    from paper_2411_15707_b200 import nimbus
    return nimbus.from_numpy_u64(a, DEV)


@pytest.mark.parametrize("N,m,n,kq,nq", [(64, 16, 20, 12, 1), (256, 130, 100, 33, 2), (128, 300, 128, 7, 1)])
def test_ell64_parity(nb, oracle, N, m, n, kq, nq):
    """ell = 64, q = 5 x 31-bit primes, 3-limb output: Enc(W), the
    output ciphertexts and R bit-exact against the Python-integer oracle
    (oracle/wide.py); decryption gives X.W - R mod 2^64 in every slot."""
    from oracle import wide
    L, ell, L_out = 5, 64, 3
    seed = 0x6464 + N + m
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    pr = [int(p) for p in nb.nimbus_ctx_primes(ctx)]
    assert pr == [int(p) for p in oracle.primes(N, L)]
    sk = nb.nimbus_keygen(ctx, seed)
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, m, n, ell)
    X = ni.gen_X(seed ^ 0xA5, kq * nq, m, ell)
    w = nb.nimbus_encrypt_weights_u64(ctx, sk, _dev_u64(W), seed)
    E = wide.encrypt_rows(N, L, pr, ell, s, W, seed)
    assert (u32(nb.nimbus_encw_export(w)) == E).all()
    ws = nb.alloc_workspace(ctx, w, kq * nq)
    cts, R = nb.alloc_outputs_u64(ctx, w, kq, nq)
    nb.nimbus_cop_matmul_u64(ctx, w, _dev_u64(X), kq, nq, seed, cts, R, ws)
    nb.nimbus_sync(ctx)
    cts_o, R_o = wide.cop_matmul(N, L, L_out, pr, ell, E, X, n, kq, nq, seed)
    assert (u32(cts) == cts_o).all()
    assert (_u64(R) == R_o).all()
    Z, _ = nb.nimbus_decrypt_u64(ctx, sk, cts, kq, nq, n)
    Y = matmul_mod_t(X, W, ell)
    with np.errstate(over="ignore"):
        assert (_u64(Z) == Y - R_o).all()


@pytest.mark.parametrize("k,m,n", [(1, 1, 1), (33, 130, 100), (128, 768, 768), (70, 3072, 129), (200, 300, 260)])
def test_plain_matmul_u64_parity(nb, oracle, k, m, n):
    """Server step 5's W<X>_s at the paper's t = 2^64: nimbus_plain_matmul_u64
    (8 byte slices, the 36 slice pairs with shift < 64 on the int8 tensor cores) equals the oracle's
    uint64 product bit for bit, with and without the added term; ragged k / m / n tiles, m up to 3072."""
    from oracle import wide
    ctx = nb.nimbus_ctx_create(8192, 5, 64, 3)
    W = ni.gen_W(31 + m, m, n, 64)
    X = ni.gen_X(32 + k, k, m, 64)
    w = nb.nimbus_plain_weights_u64(ctx, _dev_u64(W))
    Y = nb.nimbus_plain_matmul_u64(ctx, w, _dev_u64(X))
    want = wide.plain_matmul64(X, W)
    assert (_u64(Y) == want).all()
    A = ni.gen_X(33, k, n, 64)
    Y2 = nb.nimbus_plain_matmul_u64(ctx, w, _dev_u64(X), add=_dev_u64(A))
    with np.errstate(over="ignore"):
        assert (_u64(Y2) == want + A).all()
    # all-ones operands: every carry of every slice product
    Xf = np.full((5, m), (1 << 64) - 1, np.uint64)
    Wf = np.full((m, n), (1 << 64) - 1, np.uint64)
    wf = nb.nimbus_plain_weights_u64(ctx, _dev_u64(Wf))
    assert (_u64(nb.nimbus_plain_matmul_u64(ctx, wf, _dev_u64(Xf))) == wide.plain_matmul64(Xf, Wf)).all()


@pytest.mark.parametrize("N,m,n,kq,nq", [(64, 16, 20, 12, 1), (256, 130, 100, 33, 2)])
def test_server_output_u64_parity_and_shares(nb, oracle, N, m, n, kq, nq):
    """Alg. 1 end to end at t = 2^64 on the GPU: client COP (nimbus_cop_matmul_u64) + server
    step 5 (nimbus_server_output_u64).  <Y>_s equals the wide oracle's bit for bit, and
    <Y>_s + R = (X_s + X_c).W mod 2^64."""
    from oracle import wide
    L, ell, L_out = 5, 64, 3
    seed = 0x5E64 + N + m
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    pr = [int(p) for p in nb.nimbus_ctx_primes(ctx)]
    sk = nb.nimbus_keygen(ctx, seed)
    s = oracle.keygen(N, seed)
    W = ni.gen_W(seed, m, n, ell)
    Xc = ni.gen_X(seed ^ 0xA5, kq * nq, m, ell)
    Xs = ni.gen_X(seed ^ 0x5A, kq * nq, m, ell)
    w = nb.nimbus_encrypt_weights_u64(ctx, sk, _dev_u64(W), seed)
    ws = nb.alloc_workspace(ctx, w, kq * nq)
    cts, R = nb.alloc_outputs_u64(ctx, w, kq, nq)
    nb.nimbus_cop_matmul_u64(ctx, w, _dev_u64(Xc), kq, nq, seed, cts, R, ws)
    pw = nb.nimbus_plain_weights_u64(ctx, _dev_u64(W))
    Ys = nb.nimbus_server_output_u64(ctx, sk, pw, _dev_u64(Xs), cts, kq, nq)
    nb.nimbus_sync(ctx)
    want = wide.server_output(N, L_out, pr, ell, s, u32(cts), Xs, W, kq, nq)
    assert (_u64(Ys) == want).all()
    with np.errstate(over="ignore"):
        assert (_u64(Ys) + _u64(R) == wide.plain_matmul64(Xc + Xs, W)).all()


def test_ell64_full_size_decrypts(nb, oracle):
    """C4's FFN-down shape at the paper's ell = 64 (N = 8192, 5 limbs, m = 3072,
    k = 128): every output slot decrypts to X.W - R mod 2^64 (valid slots) or
    -r (invalid ones)."""
    N, L, ell, L_out, m, n, kq = 8192, 5, 64, 3, 3072, 768, 128
    seed = ni.seed_mm(4)
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, seed)
    W = ni.gen_W(seed, m, n, ell)
    X = ni.gen_X(seed, kq, m, ell)
    w = nb.nimbus_encrypt_weights_u64(ctx, sk, _dev_u64(W), seed)
    ws = nb.alloc_workspace(ctx, w, kq)
    cts, R = nb.alloc_outputs_u64(ctx, w, kq, 1)
    nb.nimbus_cop_matmul_u64(ctx, w, _dev_u64(X), kq, 1, seed, cts, R, ws)
    Z, M = nb.nimbus_decrypt_u64(ctx, sk, cts, kq, 1, n, want_full=True)
    Y = matmul_mod_t(X, W, ell)
    Rn = _u64(R)
    with np.errstate(over="ignore"):
        assert (_u64(Z) == Y - Rn).all()
    Mn = _u64(M)
    Rr = N // n
    for tg in range(Mn.shape[0]):
        rows = min(Rr, kq - tg * Rr)
        mask = ni.prg_words(seed, 6, tg * N, N)
        with np.errstate(over="ignore"):
            assert (Mn[tg][rows * n:] == (np.uint64(0) - mask[rows * n:])).all()
    # the ciphertext bytes themselves, at the full shape: Enc(W) in full and 64 sampled output
    # coefficients (both components, all 3 output limbs) against the wide (Python-integer) oracle
    from oracle import wide
    pr = [int(p) for p in nb.nimbus_ctx_primes(ctx)]
    E = wide.encrypt_rows(N, L, pr, ell, oracle.keygen(N, seed), W, seed)
    assert (u32(nb.nimbus_encw_export(w)) == E).all()
    rng = np.random.default_rng(64)
    nct = cts.shape[1]
    st = rng.integers(0, nct, 64)
    sJ = rng.integers(0, N, 64)
    st[:4], sJ[:4] = [0, nct - 1, nct - 1, 5], [0, N - 1, (kq - (nct - 1) * Rr) * n, n - 1]
    want = wide.cop_matmul_sampled(N, L, L_out, pr, ell, E, X, n, kq, 1, seed, np.zeros(64, int), st, sJ)
    g = u32(cts)
    assert (np.stack([g[0, st[i], :, :, sJ[i]] for i in range(64)]) == want).all()


def test_width_guards(nb):
    """32-bit entry points refuse ell > 32 contexts and the _u64 ones ell <= 32."""
    c64 = nb.nimbus_ctx_create(256, 5, 64, 3)
    sk = nb.nimbus_keygen(c64, 1)
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_encrypt_weights(c64, sk, dev_u32(ni.gen_W(1, 4, 4, 16)), 1)
    assert e.value.status == -1
    c16 = nb.nimbus_ctx_create(256, 2, 16, 1)
    sk16 = nb.nimbus_keygen(c16, 1)
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_encrypt_weights_u64(c16, sk16, _dev_u64(ni.gen_W(1, 4, 4, 64)), 1)
    assert e.value.status == -1
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_ctx_create(256, 5, 64, 4)          # q' would exceed 2^95
    assert e.value.status == -1


# ------------------------------------------------------------------ seeded random shapes
def _fuzz_cases(count=None, seed=None):
    """24 seeded cases by default; NIMBUS_FUZZ_CASES=<count> (and NIMBUS_FUZZ_SEED) for a
    longer soak, which also draws N = 2048 / 4096."""
    import os
    count = int(os.environ.get("NIMBUS_FUZZ_CASES", "24")) if count is None else count
    seed = int(os.environ.get("NIMBUS_FUZZ_SEED", "2024")) if seed is None else seed
    Ns = [64, 128, 256, 512, 1024] + ([2048, 4096] if count > 24 else [])
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        N = int(rng.choice(Ns))
        ell = int(rng.choice([4, 8, 12, 16, 24, 32]))
        L = 2 if ell <= 16 else 3
        L_out = 1 if ell <= 16 else 2
        n = int(rng.integers(1, N + 1))
        m = int(rng.integers(1, 400))
        kq = int(rng.integers(1, 140))
        nq = int(rng.integers(1, 3))
        out.append((N, L, ell, L_out, m, n, kq, nq))
    return out


def _fuzz_cases_large_k(count=None, seed=None):
    """Seeded shapes for the NIMBUS_FLAG_LARGE_K layout (128-column tiles) at ell in (8, 32]:
    half of them with n a multiple of 128 and enough rows for the packed contraction.
    16 cases by default; NIMBUS_FUZZ_LK_CASES=<count> (and NIMBUS_FUZZ_LK_SEED) for a soak,
    which also draws N = 4096."""
    import os
    count = int(os.environ.get("NIMBUS_FUZZ_LK_CASES", "16")) if count is None else count
    seed = int(os.environ.get("NIMBUS_FUZZ_LK_SEED", "31337")) if seed is None else seed
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        N = int(rng.choice([256, 512, 1024, 2048] + ([4096] if count > 16 else [])))
        ell = int(rng.choice([12, 16, 24, 32]))
        L, L_out = (3, 1) if ell <= 16 else (3, 2)
        if i % 2 == 0:
            n = 128 * int(rng.integers(1, N // 128 + 1))
            R = N // n
            kq = int(rng.integers(48 * R // 2 + 1, 48 * R + 200))
            nq = 2
        else:
            n = int(rng.integers(1, N + 1))
            kq = int(rng.integers(1, 300))
            nq = int(rng.integers(1, 3))
        m = int(rng.integers(1, 700))
        out.append((N, L, ell, L_out, m, n, kq, nq))
    return out


@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,nq", _fuzz_cases_large_k())
def test_random_shapes_large_k_parity(nb, oracle, N, L, ell, L_out, m, n, kq, nq):
    """Seeded random shapes on the transposed layout (NIMBUS_FLAG_LARGE_K): the packed
    contraction at S_x = 2 and 4 where it applies, the transposed row-wise kernel otherwise;
    bit-exact vs the oracle and decrypting to X.W - R mod t."""
    try:
        c = Case(nb, oracle, N, L, ell, L_out, m, n, kq, nq, seed=0xA00 + m * 7 + n, flags=nb.FLAG_LARGE_K)
        cts, R = c.run()
    except nb.NimbusError as e:
        assert e.status == -4
        return
    cts_o, R_o = c.oracle_out()
    assert (u32(cts) == cts_o).all() and (u32(R) == R_o).all()
    c.check_decrypt(cts, R)


@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,nq", _fuzz_cases())
def test_random_shapes_parity(nb, oracle, N, L, ell, L_out, m, n, kq, nq):
    """Seeded random (N, ell, m, n, k, queries): output ciphertexts and R bit-exact
    vs the oracle, every slot decrypting to X.W - R mod t.  Shapes the noise bound
    refuses must be refused with NIMBUS_ENOISE, consistently at encrypt or matmul."""
    try:
        c = Case(nb, oracle, N, L, ell, L_out, m, n, kq, nq, seed=0xF00 + m * 7 + n)
    except nb.NimbusError as e:
        assert e.status == -4
        return
    try:
        cts, R = c.run()
    except nb.NimbusError as e:
        assert e.status == -4
        return
    cts_o, R_o = c.oracle_out()
    assert (u32(cts) == cts_o).all() and (u32(R) == R_o).all()
    c.check_decrypt(cts, R)


def test_ell64_batch_and_streamed_match_single(nb, oracle):
    """ell = 64 through the batched (pack on the side stream) and the streamed
    (Enc(W) from pinned host memory) calls: the same bytes as job-by-job
    nimbus_cop_matmul_u64."""
    N, L, ell, L_out = 256, 5, 64, 3
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 9)
    shapes = [(33, 130, 100, 2), (7, 300, 128, 1), (64, 64, 256, 1)]
    jobs, ref = [], []
    for i, (kq, m, n, nq) in enumerate(shapes):
        w = nb.nimbus_encrypt_weights_u64(ctx, sk, _dev_u64(ni.gen_W(70 + i, m, n, ell)), 70 + i)
        X = _dev_u64(ni.gen_X(80 + i, kq * nq, m, ell))
        ws = nb.alloc_workspace(ctx, w, kq * nq)
        c0, R0 = nb.alloc_outputs_u64(ctx, w, kq, nq)
        nb.nimbus_cop_matmul_u64(ctx, w, X, kq, nq, 90 + i, c0, R0, ws)
        ref.append((c0, R0))
        cts, R = nb.alloc_outputs_u64(ctx, w, kq, nq)
        jobs.append(dict(encw=w, X=X, k_per_query=kq, n_queries=nq, mask_seed=90 + i, cts=cts, R=R))
    wsb = torch.empty(nb.nimbus_cop_workspace_size_batch_u64(ctx, jobs), dtype=torch.uint8, device=DEV)
    nb.nimbus_cop_matmul_batch_u64(ctx, jobs, wsb)
    nb.nimbus_sync(ctx)
    for j, (c0, R0) in zip(jobs, ref):
        assert torch.equal(j["cts"], c0) and torch.equal(j["R"], R0)
        j["cts"].zero_()
        j["R"].zero_()
    for j in jobs:
        nb.nimbus_encw_offload(j["encw"])
    ws = torch.empty(max(nb.nimbus_cop_workspace_size(ctx, j["encw"], j["k_per_query"] * j["n_queries"])
                         for j in jobs), dtype=torch.uint8, device=DEV)
    stage = torch.empty(nb.nimbus_cop_stage_size_u64(ctx, jobs), dtype=torch.uint8, device=DEV)
    nb.nimbus_cop_matmul_streamed_u64(ctx, jobs, ws, stage)
    nb.nimbus_sync(ctx)
    for j, (c0, R0) in zip(jobs, ref):
        assert torch.equal(j["cts"], c0) and torch.equal(j["R"], R0)


def test_store_file_roundtrip_and_corruption(nb, oracle, tmp_path):
    """Enc(W) store file: save -> load gives the same
    canonical Enc(W) and the same matmul outputs; a flipped payload byte, a
    truncated file or a context with other parameters are refused with NIMBUS_EIO."""
    ctx = nb.nimbus_ctx_create(1024, 2, 16, 1)
    sk = nb.nimbus_keygen(ctx, 3)
    W = ni.gen_W(5, 200, 300, 16)
    w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(W), 5)
    path = str(tmp_path / "encw.nimbus")
    nb.nimbus_encw_save(w, path)
    w2 = nb.nimbus_encw_load(ctx, path)
    assert (w2.m, w2.n) == (200, 300)
    assert torch.equal(nb.nimbus_encw_export(w2), nb.nimbus_encw_export(w))
    X = dev_u32(ni.gen_X(6, 20, 200, 16))
    ws = nb.alloc_workspace(ctx, w, 20)
    c1, R1 = nb.alloc_outputs(ctx, w, 20, 1)
    c2, R2 = nb.alloc_outputs(ctx, w2, 20, 1)
    nb.nimbus_cop_matmul(ctx, w, X, 20, 1, 7, c1, R1, ws)
    nb.nimbus_cop_matmul(ctx, w2, X, 20, 1, 7, c2, R2, ws)
    nb.nimbus_sync(ctx)
    assert torch.equal(c1, c2) and torch.equal(R1, R2)
    raw = open(path, "rb").read()
    bad = bytearray(raw)
    bad[100] ^= 1
    open(str(tmp_path / "flip"), "wb").write(bytes(bad))
    open(str(tmp_path / "trunc"), "wb").write(raw[:-9])
    for p in ("flip", "trunc", "missing"):
        with pytest.raises(nb.NimbusError) as e:
            nb.nimbus_encw_load(ctx, str(tmp_path / p))
        assert e.value.status == -7
    other = nb.nimbus_ctx_create(1024, 3, 16, 1)
    with pytest.raises(nb.NimbusError) as e:
        nb.nimbus_encw_load(other, path)
    assert e.value.status == -7
