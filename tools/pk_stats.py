"""Cycle accounting of the packed contraction (k_cop_pk) from the trace build
(NIMBUS_TRACE=1 python paper_2411_15707_b200/_build.py): runs one C5-shaped job list
(--layers L of the 12, default all) through nimbus_cop_matmul_batch and prints, averaged
over CTAs, where the MMA warp's and the epilogue's cycles went."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NIMBUS_LIB", "libnimbus_cop_trace.so")
import torch  # noqa: E402

import nimbus_inputs as ni  # noqa: E402
from paper_2411_15707_b200 import nimbus as nb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=12)
ap.add_argument("--config", default="5")
ap.add_argument("--projs", default="Q,K,V,O,up,down", help="projections of each layer to include")
args = ap.parse_args()
cfg = ni.CONFIGS_L16[int(args.config[0])] if args.config.endswith("l16") else ni.CONFIGS[int(args.config)]
keep = [ni._PROJ.index(p) for p in args.projs.split(",")]
ctx = nb.nimbus_ctx_create(cfg.N, cfg.L, cfg.ell, cfg.L_out, flags=nb.FLAG_LARGE_K)
sk = nb.nimbus_keygen(ctx, 1)
jobs = []
for li, pj, lay in cfg.layers[: 6 * args.layers]:
    if pj not in keep:
        continue
    seed = ni.seed_mm(cfg.cid, li, pj)
    w = nb.nimbus_encrypt_weights(ctx, sk, nb.from_numpy_u32(ni.gen_W(seed, lay.m, lay.n, cfg.ell), "cuda"), seed)
    cts, R = nb.alloc_outputs(ctx, w, lay.k_per_query, lay.n_queries)
    jobs.append(dict(encw=w, X=nb.from_numpy_u32(ni.gen_X(seed, lay.k, lay.m, cfg.ell), "cuda"),
                     k_per_query=lay.k_per_query, n_queries=lay.n_queries, mask_seed=seed, cts=cts, R=R))
ws = torch.empty(nb.nimbus_cop_workspace_size_batch(ctx, jobs), dtype=torch.uint8, device="cuda")
for _ in range(2):
    nb.nimbus_cop_matmul_batch(ctx, jobs, ws)
torch.cuda.synchronize()
st = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
lib = nb.lib()
lib.nimbus_pk_stats_set(ctypes.c_void_p(st.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
nb.nimbus_cop_matmul_batch(ctx, jobs, ws)
e1.record()
torch.cuda.synchronize()
lib.nimbus_pk_stats_set(ctypes.c_void_p(0))
s = st.view(148, 16).double().mean(0).tolist()
tot = s[3]
print(f"kernel {nb.nimbus_last_contraction(ctx)}  pass {e0.elapsed_time(e1):.2f} ms (trace build)  units/CTA {s[7]:.1f}")
print(f"MMA warp: total {tot/1e6:.1f} Mcyc | wait accum {s[0]/tot:.1%} | wait X {s[1]/tot:.1%} | wait E {s[2]/tot:.1%} | "
      f"issuing {(tot - s[0] - s[1] - s[2])/tot:.1%}")
print(f"epilogue (per warp): drains {s[4]/8/tot:.1%} (of which TMEM loads {s[11]/8/tot:.1%}) | finalize {s[5]/8/tot:.1%} | "
      f"wait accum {s[6]/8/tot:.1%} | prefetch/flags {s[8]/8/tot:.1%}")
u = s[7]
print(f"per unit (avg over {u:.0f}): MMA wait accum {s[0]/u:.0f} cyc, drain {s[4]/8/u:.0f} cyc (loads {s[11]/8/u:.0f}), "
      f"finalize {s[5]/8/u:.0f} cyc, MMA total {tot/u:.0f} cyc")
uo = max(s[14], 1.0)
print(f"finalize split (per warp): output passes {s[12]/8/uo:.0f} cyc/unit over {uo:.0f} units, dropped-limb passes "
      f"{s[13]/8/max(u - uo, 1):.0f} cyc/unit + fence/flag {(s[5] - s[12] - s[13])/8/max(u - uo, 1):.0f}")
print(f"producer: waiting for free E slots {s[9]/tot:.1%} | X slots {s[10]/tot:.1%}")
