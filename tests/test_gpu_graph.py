"""CUDA-graph capture of the online path: nimbus_cop_matmul (the PDL chain
slice -> contraction -> pack) and nimbus_cop_matmul_batch (pack on the
library's side stream, joined by events) contain no allocation and no host
synchronisation, so a caller can capture them once and replay them; each replay
must give the bytes a direct call gives for the inputs in the captured buffers
at replay time."""
import pytest
import torch

import nimbus_inputs as ni
from test_gpu_parity import dev_u32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_15707_b200 import nimbus
    nimbus.lib()
    return nimbus


@pytest.mark.parametrize("N,L,ell,L_out,m,n,kq,nq", [(4096, 2, 16, 1, 768, 768, 128, 1),     # C2 shape
                                                     (8192, 3, 32, 2, 300, 1000, 70, 3),    # ell = 32, streaming
                                                     (4096, 2, 16, 1, 64, 64, 16, 1)])      # C1 shape
def test_graph_replay_matches_direct(nb, N, L, ell, L_out, m, n, kq, nq):
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 31)
    w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(31, m, n, ell)), 31)
    Xs = [dev_u32(ni.gen_X(40 + i, kq * nq, m, ell)) for i in range(3)]
    ws = nb.alloc_workspace(ctx, w, kq * nq)
    ref = []
    for X in Xs:
        c, R = nb.alloc_outputs(ctx, w, kq, nq)
        nb.nimbus_cop_matmul(ctx, w, X, kq, nq, 77, c, R, ws)
        ref.append((c, R))
    torch.cuda.synchronize()
    Xbuf = Xs[0].clone()
    cts, R = nb.alloc_outputs(ctx, w, kq, nq)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):                       # warm-up on the capture stream
        nb.nimbus_cop_matmul(ctx, w, Xbuf, kq, nq, 77, cts, R, ws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        nb.nimbus_cop_matmul(ctx, w, Xbuf, kq, nq, 77, cts, R, ws, stream=s)
    for rep in range(6):
        i = rep % 3
        Xbuf.copy_(Xs[i])
        cts.zero_()
        R.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(cts, ref[i][0]) and torch.equal(R, ref[i][1]), f"replay {rep}"


def test_graph_batch_replay(nb):
    """A captured job list (side-stream packs joined by events) replays to the same bytes."""
    N, L, ell, L_out = 4096, 2, 16, 1
    ctx = nb.nimbus_ctx_create(N, L, ell, L_out)
    sk = nb.nimbus_keygen(ctx, 32)
    shapes = [(128, 768, 768, 1), (64, 300, 700, 2), (128, 768, 3072, 1)]
    jobs, ref = [], []
    for i, (kq, m, n, nq) in enumerate(shapes):
        w = nb.nimbus_encrypt_weights(ctx, sk, dev_u32(ni.gen_W(50 + i, m, n, ell)), 50 + i)
        X = dev_u32(ni.gen_X(60 + i, kq * nq, m, ell))
        c0, R0 = nb.alloc_outputs(ctx, w, kq, nq)
        nb.nimbus_cop_matmul(ctx, w, X, kq, nq, 70 + i, c0, R0, nb.alloc_workspace(ctx, w, kq * nq))
        ref.append((c0, R0))
        cts, R = nb.alloc_outputs(ctx, w, kq, nq)
        jobs.append(dict(encw=w, X=X, k_per_query=kq, n_queries=nq, mask_seed=70 + i, cts=cts, R=R))
    wsb = torch.empty(nb.nimbus_cop_workspace_size_batch(ctx, jobs), dtype=torch.uint8, device="cuda:0")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        nb.nimbus_cop_matmul_batch(ctx, jobs, wsb, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        nb.nimbus_cop_matmul_batch(ctx, jobs, wsb, stream=s)
    for rep in range(3):
        for j in jobs:
            j["cts"].zero_()
            j["R"].zero_()
        g.replay()
        torch.cuda.synchronize()
        for j, (c0, R0) in zip(jobs, ref):
            assert torch.equal(j["cts"], c0) and torch.equal(j["R"], R0)
