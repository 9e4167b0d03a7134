"""Host-side multi-rank logic of bench.py, run as world_size 2 over gloo on
CPU: independent per-rank queries (weak scaling, no data-path collective),
max-over-ranks timing, and the whole-job value."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import nimbus_inputs as ni
    # each rank draws its own X for the same weight matrix
    X = ni.gen_X(bench.rank_x_seed(ni.seed_mm(2), rank), 4, 8, 16)
    gathered = [torch.zeros(32, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(X.astype("int64").ravel()))
    # per-rank step times: the job time is the max over ranks
    local_ms = 1.0 + rank
    job_ms = bench.max_over_ranks(local_ms, world, "cpu")
    out[rank] = (job_ms, [g.tolist() for g in gathered],
                 bench.weak_value(1e9, world, job_ms))
    dist.destroy_process_group()


def test_weak_scaling_logic_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    (m0, g0, v0), (m1, g1, v1) = out[0], out[1]
    assert m0 == m1 == 2.0                      # max over ranks
    assert g0 == g1 and g0[0] != g0[1]          # independent queries per rank
    assert v0 == v1 == pytest.approx(2 * 1e9 / 2e-3)   # all ranks' units / max time


def test_single_rank_is_identity():
    import bench
    assert bench.max_over_ranks(3.5, 1, "cpu") == 3.5
    assert bench.rank_x_seed(123, 0) == 123
