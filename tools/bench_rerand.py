"""Cost of circuit privacy (reading 26) on the GPU for one config:
the online call with and without the public-key zero encryptions added in the
pack (nimbus_cop_matmul_rr vs nimbus_cop_matmul), and the offline
nimbus_rerand_prepare.  CUDA events on the launching stream, warm; one JSON line.

  python tools/bench_rerand.py --config 2 --steps 300
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import nimbus_inputs as ni
from paper_2411_15707_b200 import nimbus as nb


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    args = ap.parse_args()
    cfg = ni.CONFIGS[int(args.config)]
    li, pj, lay = cfg.layers[0]
    seed = ni.seed_mm(cfg.cid, li, pj)
    dev = "cuda:0"
    ctx = nb.nimbus_ctx_create(cfg.N, cfg.L, cfg.ell, cfg.L_out)
    sk = nb.nimbus_keygen(ctx, cfg.seed_cfg)
    pk = nb.nimbus_keygen_pk(ctx, sk, cfg.seed_cfg ^ 1)
    w = nb.nimbus_encrypt_weights(ctx, sk, nb.from_numpy_u32(ni.gen_W(seed, lay.m, lay.n, cfg.ell), dev), seed)
    X = nb.from_numpy_u32(ni.gen_X(seed, lay.k, lay.m, cfg.ell), dev)
    kq, nq = lay.k_per_query, lay.n_queries
    ws = nb.alloc_workspace(ctx, w, lay.k)
    cts, R = nb.alloc_outputs(ctx, w, kq, nq)
    F = nb.nimbus_rerand_flood_max(ctx, w, kq)
    zero = nb.alloc_zero(ctx, w, kq, nq)
    t_prep = timed(lambda: nb.nimbus_rerand_prepare(ctx, pk, w, kq, nq, seed, F, zero), 20, 2)
    # alternate the two calls in blocks (min per call): a tensor-bound config heats the
    # GPU into its power cap, so a single back-to-back pair would favour the first
    t_plain = t_rr = float("inf")
    for _ in range(4):
        t_plain = min(t_plain, timed(lambda: nb.nimbus_cop_matmul(ctx, w, X, kq, nq, seed, cts, R, ws),
                                     args.steps // 4, args.warmup))
        t_rr = min(t_rr, timed(lambda: nb.nimbus_cop_matmul_rr(ctx, w, X, kq, nq, seed, zero, cts, R, ws),
                               args.steps // 4, args.warmup))
    print(json.dumps({"workload": f"{cfg.name}: {zero.shape[0]} output ciphertexts, flood bits {F}",
                      "cop_matmul_us": t_plain, "cop_matmul_rr_us": t_rr, "rr_overhead_us": t_rr - t_plain,
                      "rerand_prepare_us": t_prep, "zero_bytes": zero.numel() * 4, "warm_l2": True}))


if __name__ == "__main__":
    main()
