"""Out-of-bounds write checks (compute-sanitizer is not available on the GPU
pool): every output buffer and workspace the C ABI writes is carved out of a
larger device buffer pre-filled with a sentinel, with guard regions before and
after it; after each call the guards must be intact, the inputs unchanged, and
the results equal to the same call on plain allocations.  Shapes are ragged in
every dimension so the tail tiles, half k-block pairs, partial packed
ciphertexts and the last query are exercised, for every contraction kernel
(resident-X with either ring, streaming, transposed, ell = 64, CUDA cores) and
the server-side calls."""
import numpy as np
import pytest
import torch

import nimbus_inputs as ni
from test_gpu_parity import dev_u32, u32

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
GUARD = 8192          # bytes of guard on each side
SENT = 0x5A           # sentinel byte


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_15707_b200 import nimbus
    nimbus.lib()
    return nimbus


class Arena:
    """Guarded device allocations: view(shape, dtype) returns a contiguous tensor
    whose bytes sit between two sentinel-filled guard regions."""

    def __init__(self):
        self.bufs = []

    def view(self, shape, dtype):
        nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        buf = torch.full((GUARD + nbytes + GUARD,), SENT, dtype=torch.uint8, device=DEV)
        self.bufs.append(buf)
        return buf[GUARD:GUARD + nbytes].view(dtype).view(shape)

    def check(self):
        torch.cuda.synchronize()
        for i, b in enumerate(self.bufs):
            assert bool((b[:GUARD] == SENT).all()), f"buffer {i}: write before its start"
            assert bool((b[-GUARD:] == SENT).all()), f"buffer {i}: write past its end"


def _xw_minus(X, W, R, ell):
    """(X W - R) mod 2^ell, exact: uint64 arithmetic wraps mod 2^64 and 2^ell divides 2^64."""
    with np.errstate(over="ignore"):
        v = X.astype(np.uint64) @ W.astype(np.uint64) - R.astype(np.uint64)
    return v & np.uint64((1 << ell) - 1) if ell < 64 else v


def _matmul_guarded(nb, ctx, w, X, kq, nq, seed, wide=False):
    """nimbus_cop_matmul[_u64] into guarded cts / R / workspace; returns (cts, R)."""
    A = Arena()
    nct = nb.nimbus_cop_out_count(ctx, kq, w.n)
    cts = A.view((nq, nct, 2, ctx.L_out, ctx.N), torch.int32)
    R = A.view((nq * kq, w.n), torch.int64 if wide else torch.int32)
    ws = A.view((nb.nimbus_cop_workspace_size(ctx, w, kq * nq),), torch.uint8)
    X0 = X.clone()
    (nb.nimbus_cop_matmul_u64 if wide else nb.nimbus_cop_matmul)(ctx, w, X, kq, nq, seed, cts, R, ws)
    A.check()
    assert torch.equal(X, X0), "input X modified"
    # the same call on plain allocations
    c2, R2 = (nb.alloc_outputs_u64 if wide else nb.alloc_outputs)(ctx, w, kq, nq)
    ws2 = nb.alloc_workspace(ctx, w, kq * nq)
    (nb.nimbus_cop_matmul_u64 if wide else nb.nimbus_cop_matmul)(ctx, w, X, kq, nq, seed, c2, R2, ws2)
    torch.cuda.synchronize()
    assert torch.equal(cts, c2) and torch.equal(R, R2)
    return cts, R


@pytest.mark.parametrize("env,N,L,ell,L_out,m,n,kq,nq,impl", [
    ({}, 4096, 2, 16, 1, 300, 1000, 70, 1, 0),                      # resident-X, 3-slot ring
    ({"NIMBUS_RES": "2"}, 4096, 2, 16, 1, 700, 77, 33, 3, 0),       # resident-X, deep ring, 6 k-blocks
    ({"NIMBUS_NO_RESIDENT": "1"}, 4096, 2, 16, 1, 129, 500, 100, 1, 0),   # streaming, ell = 16
    ({}, 4096, 2, 16, 1, 1000, 300, 150, 2, 0),                     # streaming (k > 128, m > 768)
    ({}, 8192, 3, 32, 2, 300, 1000, 70, 3, 0),                      # streaming, ell = 32, 2 output limbs
    ({"NIMBUS_TRANSPOSED": "1"}, 8192, 3, 32, 2, 257, 129, 65, 2, 0),   # transposed, ell = 32
    ({"NIMBUS_TRANSPOSED": "1"}, 1024, 3, 16, 1, 257, 129, 65, 2, 0),   # transposed, ell = 16 (S_x = 2)
    ({"NIMBUS_TRANSPOSED": "1"}, 1024, 3, 32, 2, 200, 128, 300, 2, 0),  # packed contraction, S_x = 4
    ({"NIMBUS_TRANSPOSED": "1"}, 1024, 3, 16, 1, 200, 128, 300, 2, 0),  # packed contraction, S_x = 2
    ({"NIMBUS_CLUSTER": "2", "NIMBUS_NO_RESIDENT": "1"}, 4096, 2, 16, 1, 200, 100, 130, 1, 0),
    ({}, 4096, 2, 16, 1, 300, 1000, 70, 1, 1),                      # CUDA-core ablation
    ({}, 4096, 2, 16, 1, 300, 2051, 60, 2, 0),                      # fused R = 1 epilogue, ragged R tail
    ({}, 4096, 2, 16, 1, 300, 3072, 128, 1, 0),                     # fused R = 1 epilogue, uint4 R stores
])
def test_cop_matmul_no_oob(nb, monkeypatch, env, N, L, ell, L_out, m, n, kq, nq, impl):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out, impl)
    sk = nb.nimbus_keygen(ctx, 3)
    w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(3, m, n, ell)), 3)
    X = dev_u32(ni.gen_X(4, kq * nq, m, ell))
    cts, R = _matmul_guarded(nb, ctx, w, X, kq, nq, 5)
    # decrypt into guarded Z / M (the verification path)
    A = Arena()
    Z = A.view((nq * kq, n), torch.int32)
    nct = nb.nimbus_cop_out_count(ctx, kq, n)
    M = A.view((nq * nct, N), torch.int32)
    nb._check(nb.lib().nimbus_decrypt(ctx.ptr, sk.ptr, nb._ptr(cts), kq, n, nq, nb._ptr(Z), nb._ptr(M),
                                      nb._stream(None)), ctx)
    A.check()
    Xn, Wn = ni.gen_X(4, kq * nq, m, ell), ni.gen_W(3, m, n, ell)
    assert (u32(Z) == _xw_minus(Xn, Wn, u32(R), ell)).all()


def test_ell64_no_oob(nb):
    N, L, ell, L_out, m, n, kq, nq = 256, 5, 64, 3, 130, 100, 33, 2
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 9)
    from test_gpu_parity import _dev_u64
    w = nb.nimbus_encrypt_weights_u64(ctx, sk, _dev_u64(ni.gen_W(70, m, n, ell)), 70)
    X = _dev_u64(ni.gen_X(80, kq * nq, m, ell))
    cts, R = _matmul_guarded(nb, ctx, w, X, kq, nq, 90, wide=True)
    A = Arena()
    Z = A.view((nq * kq, n), torch.int64)
    nb._check(nb.lib().nimbus_decrypt_u64(ctx.ptr, sk.ptr, nb._ptr(cts), kq, n, nq, nb._ptr(Z), None,
                                          nb._stream(None)), ctx)
    A.check()
    Xn, Wn = ni.gen_X(80, kq * nq, m, ell), ni.gen_W(70, m, n, ell)
    assert (nb.to_numpy_u64(Z) == _xw_minus(Xn, Wn, nb.to_numpy_u64(R), ell)).all()


def test_accumulate_pack_batch_host_no_oob(nb):
    """cop_accumulate / cop_pack halves, the batched call and the pipelined host
    batch, each into guarded buffers."""
    N, L, ell, L_out, m, n, kq, nq = 4096, 2, 16, 1, 520, 700, 45, 2
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 11)
    w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(11, m, n, ell)), 11)
    X = dev_u32(ni.gen_X(12, kq * nq, m, ell))
    ref_c, ref_R = nb.alloc_outputs(ctx, w, kq, nq)
    nb.nimbus_cop_matmul(ctx, w, X, kq, nq, 13, ref_c, ref_R, nb.alloc_workspace(ctx, w, kq * nq))
    A = Arena()
    Cg = A.view((kq * nq, 2, L, N), torch.int32)
    ws = A.view((nb.nimbus_cop_workspace_size(ctx, w, kq * nq),), torch.uint8)
    nb.nimbus_cop_accumulate(ctx, w, X, ws, C_out=Cg)
    A.check()
    nct = nb.nimbus_cop_out_count(ctx, kq, n)
    cts = A.view((nq, nct, 2, L_out, N), torch.int32)
    R = A.view((nq * kq, n), torch.int32)
    nb._check(nb.lib().nimbus_cop_pack(ctx.ptr, nb._ptr(Cg), kq, nq, n, 13, nb._ptr(cts), nb._ptr(R),
                                       nb._stream(None)), ctx)
    A.check()
    assert torch.equal(cts, ref_c) and torch.equal(R, ref_R)
    # batched call: two jobs, guarded outputs and workspace
    jobs = []
    for i in range(3):
        jobs.append(dict(encw=w, X=X, k_per_query=kq, n_queries=nq, mask_seed=13,
                         cts=A.view((nq, nct, 2, L_out, N), torch.int32), R=A.view((nq * kq, n), torch.int32)))
    wsb = A.view((nb.nimbus_cop_workspace_size_batch(ctx, jobs),), torch.uint8)
    nb.nimbus_cop_matmul_batch(ctx, jobs, wsb)
    A.check()
    for j in jobs:
        assert torch.equal(j["cts"], ref_c) and torch.equal(j["R"], ref_R)
    # pipelined host batch: guarded device workspace; host outputs with guards too
    hjobs, hbufs = [], []
    for i in range(5):
        hc = torch.full((GUARD + ref_c.numel() * 4 + GUARD,), SENT, dtype=torch.uint8).pin_memory()
        hr = torch.full((GUARD + ref_R.numel() * 4 + GUARD,), SENT, dtype=torch.uint8).pin_memory()
        hbufs += [hc, hr]
        hjobs.append(dict(encw=w, X=X.cpu().pin_memory(), k_per_query=kq, n_queries=nq, mask_seed=13,
                          cts=hc[GUARD:GUARD + ref_c.numel() * 4].view(torch.int32).view(ref_c.shape),
                          R=hr[GUARD:GUARD + ref_R.numel() * 4].view(torch.int32).view(ref_R.shape)))
    wsh = A.view((nb.nimbus_cop_workspace_size_host_batch(ctx, hjobs),), torch.uint8)
    nb.nimbus_cop_matmul_host_batch(ctx, hjobs, wsh)
    A.check()
    for b in hbufs:
        assert bool((b[:GUARD] == SENT).all()) and bool((b[-GUARD:] == SENT).all())
    for j in hjobs:
        assert torch.equal(j["cts"], ref_c.cpu()) and torch.equal(j["R"], ref_R.cpu())


def test_server_no_oob(nb):
    """Server step 5: plaintext GEMM and server_output into guarded buffers."""
    N, L, ell, L_out, m, n, kq, nq = 4096, 2, 16, 1, 300, 130, 70, 2
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 21)
    Wn = ni.gen_W(21, m, n, ell)
    w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(Wn), 21)
    pw = nb.nimbus_plain_weights(ctx, dev_u32(Wn))
    Xc = dev_u32(ni.gen_X(22, kq * nq, m, ell))
    Xs = dev_u32(ni.gen_X(23, kq * nq, m, ell))
    cts, R = nb.alloc_outputs(ctx, w, kq, nq)
    nb.nimbus_cop_matmul(ctx, w, Xc, kq, nq, 24, cts, R, nb.alloc_workspace(ctx, w, kq * nq))
    A = Arena()
    Y = A.view((kq * nq, n), torch.int32)
    ws = A.view((nb.nimbus_server_workspace_size(ctx, pw, kq * nq, 0),), torch.uint8)
    nb.nimbus_plain_matmul(ctx, pw, Xs, Y=Y, ws=ws)
    A.check()
    Ys = A.view((kq * nq, n), torch.int32)
    ws2 = A.view((nb.nimbus_server_workspace_size(ctx, pw, kq, nq),), torch.uint8)
    nb.nimbus_server_output(ctx, sk, pw, Xs, cts, kq, nq, Ys=Ys, ws=ws2)
    A.check()
    Xsum = ni.gen_X(22, kq * nq, m, ell).astype(np.uint64) + ni.gen_X(23, kq * nq, m, ell).astype(np.uint64)
    ref = _xw_minus(Xsum, Wn, np.zeros((kq * nq, n), np.uint64), ell)
    assert ((u32(Ys).astype(np.uint64) + u32(R).astype(np.uint64)) % np.uint64(1 << ell) == ref).all()


def test_fused_r1_misaligned_outputs(nb):
    """The fused R = 1 epilogue stores with 16-byte vectors; output buffers that are
    only 4-byte aligned must take the unfused path (same bytes), not fault."""
    N, L, ell, L_out, m, n, kq, nq = 4096, 2, 16, 1, 300, 3072, 100, 1
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 31)
    w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(31, m, n, ell)), 31)
    X = dev_u32(ni.gen_X(32, kq * nq, m, ell))
    ref_c, ref_R = nb.alloc_outputs(ctx, w, kq, nq)
    ws = nb.alloc_workspace(ctx, w, kq * nq)
    nb.nimbus_cop_matmul(ctx, w, X, kq, nq, 33, ref_c, ref_R, ws)
    bc = torch.zeros(ref_c.numel() + 1, dtype=torch.int32, device=DEV)
    br = torch.zeros(ref_R.numel() + 1, dtype=torch.int32, device=DEV)
    c4, r4 = bc[1:].view(ref_c.shape), br[1:].view(ref_R.shape)      # 4 bytes past a 16-byte boundary
    assert c4.data_ptr() % 16 == 4 and r4.data_ptr() % 16 == 4
    nb.nimbus_cop_matmul(ctx, w, X, kq, nq, 33, c4, r4, ws)
    torch.cuda.synchronize()
    assert torch.equal(c4, ref_c) and torch.equal(r4, ref_R)
