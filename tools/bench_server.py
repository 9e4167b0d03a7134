"""Time the server side of Alg. 1 step 5 on the GPU for one
config: nimbus_server_output = decrypt + unpack (K8) + X_s.W mod t (plain
tcgen05 GEMM) + add, and its two parts alone.  CUDA events on the launching
stream, warm-up first; prints one JSON line.

  python tools/bench_server.py --config 2 --steps 200
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
    return a.elapsed_time(b) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    args = ap.parse_args()
    cfg = ni.CONFIGS[int(args.config)]
    li, pj, lay = cfg.layers[0]
    seed = ni.seed_mm(cfg.cid, li, pj)
    dev = "cuda:0"
    ctx = nb.nimbus_ctx_create(cfg.N, cfg.L, cfg.ell, cfg.L_out)
    sk = nb.nimbus_keygen(ctx, cfg.seed_cfg)
    W = nb.from_numpy_u32(ni.gen_W(seed, lay.m, lay.n, cfg.ell), dev)
    encw = nb.nimbus_encrypt_weights(ctx, sk, W, seed)
    Xc = nb.from_numpy_u32(ni.gen_X(seed, lay.k, lay.m, cfg.ell), dev)
    Xs = nb.from_numpy_u32(ni.gen_X(seed + 1, lay.k, lay.m, cfg.ell), dev)
    cts, R = nb.alloc_outputs(ctx, encw, lay.k_per_query, lay.n_queries)
    nb.nimbus_cop_matmul(ctx, encw, Xc, lay.k_per_query, lay.n_queries, seed, cts, R,
                         nb.alloc_workspace(ctx, encw, lay.k))
    pw = nb.nimbus_plain_weights(ctx, W)
    ws = torch.empty(nb.nimbus_server_workspace_size(ctx, pw, lay.k_per_query, lay.n_queries), dtype=torch.uint8,
                     device=dev)
    Ys = torch.empty((lay.k, lay.n), dtype=torch.int32, device=dev)
    Z = torch.empty((lay.k, lay.n), dtype=torch.int32, device=dev)
    t_all = timed(lambda: nb.nimbus_server_output(ctx, sk, pw, Xs, cts, lay.k_per_query, lay.n_queries, Ys, ws),
                  args.steps, args.warmup)
    t_plain = timed(lambda: nb.nimbus_plain_matmul(ctx, pw, Xs, Z, Ys, ws), args.steps, args.warmup)
    t_dec = timed(lambda: nb.nimbus_decrypt(ctx, sk, cts, lay.k_per_query, lay.n_queries, lay.n), args.steps,
                  args.warmup)
    nct = nb.nimbus_cop_out_count(ctx, lay.k_per_query, lay.n) * lay.n_queries
    sx = 1 if cfg.ell <= 8 else 2 if cfg.ell <= 16 else 4
    plain_ops = 2 * lay.k * lay.m * lay.n * (sx * (sx + 1) // 2)
    print(json.dumps({
        "workload": f"{cfg.name} server step 5: Dec({nct} cts, N={cfg.N}, L_out={cfg.L_out}) + "
                    f"X_s {lay.k}x{lay.m} . W {lay.m}x{lay.n} mod 2^{cfg.ell}",
        "server_output_us": t_all * 1e3, "decrypt_unpack_us": t_dec * 1e3, "plain_matmul_us": t_plain * 1e3,
        "plain_int8_tops": plain_ops / (t_plain * 1e-3) / 1e12,
        "decrypt_cts_per_s": nct / (t_dec * 1e-3)}))


if __name__ == "__main__":
    main()
