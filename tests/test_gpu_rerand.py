"""GPU parity of the circuit-privacy path (readings 25-26; PAPER.md:602
KeyGen (sk, pk), PAPER.md:645 circuit privacy): the public key, the offline
public-key zero encryptions and the re-randomised COP output, through the C ABI,
bit-exact against the CPU oracle (oracle.keygen_pk / rerand_zero /
cop_matmul_rr, pinned in test_oracle_rerand.py), plus decryption of every slot.
"""
import numpy as np
import pytest
import torch

import nimbus_inputs as ni
from test_gpu_parity import _dev_u64, _u64, dev_u32, matmul_mod_t, u32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_15707_b200 import nimbus
    nimbus.lib()
    return nimbus


CASES = [
    # N, L, ell, L_out, m, n, kq, nq
    (4096, 2, 16, 1, 768, 768, 128, 1),      # C2 shape (R = 5, ragged last ciphertext)
    (4096, 2, 16, 1, 200, 300, 37, 2),       # ragged multi-query, R = 13
    (4096, 2, 16, 1, 128, 3072, 20, 1),      # R = 1 (C3 packing: single-row path of the pack)
    (8192, 3, 32, 2, 256, 768, 30, 1),       # ell = 32, 3 -> 2 limbs
    (8192, 3, 16, 1, 300, 1000, 17, 1),      # ell = 16 on the 3-prime ring (two limb drops)
    (4096, 3, 16, 1, 768, 768, 128, 1),      # C2 with one more limb: statistical flooding (F > 62, two words)
]


@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,nq", CASES)
def test_rerand_parity(nb, oracle, N, L, ell, L_out, m, n, kq, nq):
    seed = 0xC1C0 + N + m + n
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    pr = np.array(nb.nimbus_ctx_primes(ctx), np.uint32)
    sk = nb.nimbus_keygen(ctx, seed)
    s = nb.nimbus_sk_export(sk).cpu().numpy()
    assert (s == oracle.keygen(N, seed)).all()
    # public key (reading 25)
    pk = nb.nimbus_keygen_pk(ctx, sk, seed ^ 0x9C)
    pk_o = oracle.keygen_pk(N, L, pr, s, seed ^ 0x9C)
    assert (u32(nb.nimbus_pk_export(pk)) == pk_o).all()
    W = ni.gen_W(seed, m, n, ell)
    X = ni.gen_X(seed ^ 0xA5, kq * nq, m, ell)
    w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(W), seed)
    F = nb.nimbus_rerand_flood_max(ctx, w, kq)
    assert F >= 8
    if L == 3 and ell == 16 and N == 4096:
        # the shipped circuit-privacy parameter set: >= 40 bits of smudging over the worst-case noise
        cop = min(N // n, kq) * m * ((1 << ell) - 1) * 21.5
        assert F - np.log2(cop) >= 40, (F, np.log2(cop))
    # zero encryptions (reading 26), with the largest flooding the bound allows
    rseed = seed ^ 0xABC
    zero = nb.nimbus_rerand_prepare(ctx, pk, w, kq, nq, rseed, F)
    nct = zero.shape[0]
    z_o = oracle.rerand_zero(N, L, pr, pk_o, rseed, nct, F)
    assert (u32(zero) == z_o).all()
    # re-randomised COP output
    ws = nb.alloc_workspace(ctx, w, kq * nq)
    cts, R = nb.alloc_outputs(ctx, w, kq, nq)
    nb.nimbus_cop_matmul_rr(ctx, w, dev_u32(X), kq, nq, seed, zero, cts, R, ws)
    nb.nimbus_sync(ctx)
    E = u32(nb.nimbus_encw_export(w))
    cts_o, R_o = oracle.cop_matmul_rr(N, L, L_out, pr, ell, E, X, n, kq, nq, seed, z_o)
    assert (u32(cts) == cts_o).all()
    assert (u32(R) == R_o).all()
    # decrypts to the protocol's share: Z = X.W - R mod t in every valid slot
    Z, _ = nb.nimbus_decrypt(ctx, sk, cts, kq, nq, n)
    t = 1 << ell
    Y = matmul_mod_t(X, W, ell)
    assert (u32(Z).astype(np.uint64) == (Y + np.uint64(t) - R_o.astype(np.uint64)) % np.uint64(t)).all()
    # the a component really is re-randomised
    cts0, _ = nb.alloc_outputs(ctx, w, kq, nq)
    R0 = torch.empty_like(R)
    nb.nimbus_cop_matmul(ctx, w, dev_u32(X), kq, nq, seed, cts0, R0, ws)
    nb.nimbus_sync(ctx)
    assert (u32(cts0)[:, :, 1] != u32(cts)[:, :, 1]).mean() > 0.99
    # flooding past the bound is refused before any launch
    if F < 126:
        with pytest.raises(nb.NimbusError) as ei:
            nb.nimbus_rerand_prepare(ctx, pk, w, kq, nq, rseed, F + 1, zero)
        assert ei.value.status == -4


def test_pk_import_roundtrip(nb, oracle):
    """The exported public key (what the server sends the client) imported into a
    new context gives identical zero encryptions."""
    N, L, ell, L_out, m, n, kq = 4096, 2, 16, 1, 64, 768, 10
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 11)
    pk = nb.nimbus_keygen_pk(ctx, sk, 12)
    ctx2 = nb.nimbus_ctx_create(N, L, ell, L_out)
    pk2 = nb.nimbus_pk_import(ctx2, nb.nimbus_pk_export(pk))
    w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(1, m, n, ell)), 1)
    w2 = nb.nimbus_encw_import(ctx2, nb.nimbus_encw_export(w), n)
    z1 = nb.nimbus_rerand_prepare(ctx, pk, w, kq, 1, 77, 20)
    z2 = nb.nimbus_rerand_prepare(ctx2, pk2, w2, kq, 1, 77, 20)
    torch.cuda.synchronize()
    assert torch.equal(z1, z2)


@pytest.mark.parametrize("N,m,n,kq,nq", [(64, 16, 20, 12, 1), (256, 130, 100, 33, 2)])
def test_rerand_ell64_parity(nb, oracle, N, m, n, kq, nq):
    """The paper's ell = 64 (5 limbs, 3-limb output) with re-randomisation:
    bit-exact against the Python-integer oracle with the same zero encryptions,
    and X.W - R mod 2^64 after decryption."""
    from oracle import wide
    L, ell, L_out = 5, 64, 3
    seed = 0x6465 + N + m
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    pr = [int(p) for p in nb.nimbus_ctx_primes(ctx)]
    sk = nb.nimbus_keygen(ctx, seed)
    s = oracle.keygen(N, seed)
    pk = nb.nimbus_keygen_pk(ctx, sk, seed + 1)
    pk_o = oracle.keygen_pk(N, L, np.array(pr, np.uint32), s, seed + 1)
    assert (u32(nb.nimbus_pk_export(pk)) == pk_o).all()
    W = ni.gen_W(seed, m, n, ell)
    X = ni.gen_X(seed ^ 0xA5, kq * nq, m, ell)
    w = nb.nimbus_encrypt_weights_u64(ctx, sk, _dev_u64(W), seed)
    F = nb.nimbus_rerand_flood_max(ctx, w, kq)
    zero = nb.nimbus_rerand_prepare(ctx, pk, w, kq, nq, seed + 2, F)
    z_o = oracle.rerand_zero(N, L, np.array(pr, np.uint32), pk_o, seed + 2, zero.shape[0], F)
    assert (u32(zero) == z_o).all()
    ws = nb.alloc_workspace(ctx, w, kq * nq)
    cts, R = nb.alloc_outputs_u64(ctx, w, kq, nq)
    nb.nimbus_cop_matmul_rr_u64(ctx, w, _dev_u64(X), kq, nq, seed, zero, cts, R, ws)
    nb.nimbus_sync(ctx)
    E = wide.encrypt_rows(N, L, pr, ell, s, W, seed)
    cts_o, R_o = wide.cop_matmul(N, L, L_out, pr, ell, E, X, n, kq, nq, seed, Z0=z_o)
    assert (u32(cts) == cts_o).all()
    assert (_u64(R) == R_o).all()
    Z, _ = nb.nimbus_decrypt_u64(ctx, sk, cts, kq, nq, n)
    Y = matmul_mod_t(X, W, ell)
    with np.errstate(over="ignore"):
        assert (_u64(Z) == Y - R_o).all()
