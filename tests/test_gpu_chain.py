"""Back-to-back calls of the PDL chain (slice -> contraction -> pack, each
kernel launched while its predecessor runs): many calls
queued without host synchronisation, alternating inputs, masks and output
buffers, must each give the bytes a lone, synchronised call gives -- a race
between the pack of one call and the slice, contraction or pack of the next
would show up as a mismatch."""
import pytest
import torch

import nimbus_inputs as ni
from test_gpu_parity import dev_u32, u32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_15707_b200 import nimbus
    nimbus.lib()
    return nimbus


@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq", [(4096, 2, 16, 1, 768, 768, 128),     # C2 (R = 5)
                                                   (4096, 2, 16, 1, 768, 3072, 128),    # C3 (R = 1)
                                                   (8192, 3, 16, 1, 640, 1000, 100)])   # 3 limbs, ragged
def test_back_to_back_calls(nb, N, L, ell, L_out, m, n, kq):
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 5)
    w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(5, m, n, ell)), 5)
    Xs = [dev_u32(ni.gen_X(100 + i, kq, m, ell)) for i in range(3)]
    seeds = [7, 8, 9]
    ws = nb.alloc_workspace(ctx, w, kq)
    ref = []
    for X, sd in zip(Xs, seeds):
        c, R = nb.alloc_outputs(ctx, w, kq, 1)
        nb.nimbus_cop_matmul(ctx, w, X, kq, 1, sd, c, R, ws)
        nb.nimbus_sync(ctx)
        ref.append((u32(c), u32(R)))
    outs = [nb.alloc_outputs(ctx, w, kq, 1) for _ in range(4)]
    calls = 48
    for it in range(calls):
        j = it % 3
        c, R = outs[it % 4]
        nb.nimbus_cop_matmul(ctx, w, Xs[j], kq, 1, seeds[j], c, R, ws)
    nb.nimbus_sync(ctx)
    for it in range(calls - 4, calls):
        c, R = outs[it % 4]
        rc, rR = ref[it % 3]
        assert (u32(c) == rc).all(), f"call {it}"
        assert (u32(R) == rR).all(), f"call {it}"
    # same output buffer every call (write-after-write between consecutive packs)
    c, R = outs[0]
    for it in range(30):
        nb.nimbus_cop_matmul(ctx, w, Xs[it % 3], kq, 1, seeds[it % 3], c, R, ws)
    nb.nimbus_sync(ctx)
    assert (u32(c) == ref[29 % 3][0]).all() and (u32(R) == ref[29 % 3][1]).all()
