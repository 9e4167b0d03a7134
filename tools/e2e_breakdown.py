"""Where the end-to-end (host buffers in, host buffers out) step time of one
config goes: the host-buffer C-ABI call against its parts, each timed by wall
clock around a host-synchronising call (as bench.py's e2e), median of 50.

  python tools/e2e_breakdown.py --config 2
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import nimbus_inputs as ni
from paper_2411_15707_b200 import nimbus as nb


def wall(fn, reps=50, warm=5):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    args = ap.parse_args()
    cfg = ni.CONFIGS[int(args.config)]
    li, pj, lay = cfg.layers[0]
    seed = ni.seed_mm(cfg.cid, li, pj)
    dev = "cuda:0"
    ctx = nb.nimbus_ctx_create(cfg.N, cfg.L, cfg.ell, cfg.L_out)
    sk = nb.nimbus_keygen(ctx, cfg.seed_cfg)
    w = nb.nimbus_encrypt_weights(ctx, sk, nb.from_numpy_u32(ni.gen_W(seed, lay.m, lay.n, cfg.ell), dev), seed)
    X = nb.from_numpy_u32(ni.gen_X(seed, lay.k, lay.m, cfg.ell), dev)
    kq, nq = lay.k_per_query, lay.n_queries
    ws = nb.alloc_workspace(ctx, w, lay.k)
    cts, R = nb.alloc_outputs(ctx, w, kq, nq)
    Xh = X.cpu().pin_memory()
    ch, Rh = nb.alloc_outputs(ctx, w, kq, nq, pin=True, device="cpu")
    s = torch.cuda.current_stream()

    def host_call():
        nb.nimbus_cop_matmul_host(ctx, w, Xh, kq, nq, seed, ch, Rh, ws)

    def dev_call():
        nb.nimbus_cop_matmul(ctx, w, X, kq, nq, seed, cts, R, ws)
        s.synchronize()

    def h2d():
        X.copy_(Xh, non_blocking=True)
        s.synchronize()

    def d2h_cts():
        ch.copy_(cts, non_blocking=True)
        s.synchronize()

    def d2h_R():
        Rh.copy_(R, non_blocking=True)
        s.synchronize()

    def empty_sync():
        s.synchronize()

    # GPU-side timeline of the same sequence on one stream (events between the stages)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    seg = [[], [], []]
    for _ in range(55):
        torch.cuda.synchronize()
        ev[0].record(s)
        X.copy_(Xh, non_blocking=True)
        ev[1].record(s)
        nb.nimbus_cop_matmul(ctx, w, X, kq, nq, seed, cts, R, ws)
        ev[2].record(s)
        ch.copy_(cts, non_blocking=True)
        Rh.copy_(R, non_blocking=True)
        ev[3].record(s)
        s.synchronize()
        for i in range(3):
            seg[i].append(ev[i].elapsed_time(ev[i + 1]) * 1e3)
    gpu = {k: statistics.median(v[5:]) for k, v in zip(("h2d_X", "cop_matmul", "d2h_cts_R"), seg)}
    out = {"config": cfg.name, "gpu_timeline_us": gpu, "host_call_us": wall(host_call), "device_call_sync_us": wall(dev_call),
           "h2d_X_us": wall(h2d), "d2h_cts_us": wall(d2h_cts), "d2h_R_us": wall(d2h_R),
           "sync_only_us": wall(empty_sync),
           "bytes": {"X": Xh.numel() * 4, "cts": ch.numel() * 4, "R": Rh.numel() * 4}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
