"""Per-stage time of nimbus_cop_matmul as a function of m (contraction length)
and k, to separate fixed per-launch overhead from per-k-block cost."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import nimbus_inputs as ni
from paper_2411_15707_b200 import nimbus as nb

N, L, ell, Lo = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (4096, 2, 16, 1)))
n = 768
ctx = nb.nimbus_ctx_create(N, L, ell, Lo)
sk = nb.nimbus_keygen(ctx, 1)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for k in (128, 256, 512):
    for m in (128, 256, 512, 768, 1536, 3072):
        W = nb.from_numpy_u32(ni.gen_W(1, m, n, ell), "cuda")
        w = nb.nimbus_encrypt_weights(ctx, sk, W, 1)
        X = nb.from_numpy_u32(ni.gen_X(2, k, m, ell), "cuda")
        ws = nb.alloc_workspace(ctx, w, k)
        cts, R = nb.alloc_outputs(ctx, w, k, 1)
        for _ in range(3):
            nb.nimbus_cop_matmul(ctx, w, X, k, 1, 3, cts, R, ws)
        nb.nimbus_profile_enable(ctx, True)
        nb.nimbus_profile_read(ctx)
        for _ in range(20):
            flush.zero_()
            nb.nimbus_cop_matmul(ctx, w, X, k, 1, 3, cts, R, ws)
        ms, calls = nb.nimbus_profile_read(ctx)
        nb.nimbus_profile_enable(ctx, False)
        us = [1e3 * x / calls for x in ms]
        macs = ni.modmacs(k, m, N, L)
        ebytes = nb.nimbus_encw_bytes(w)
        print(f"k={k:4d} m={m:5d}  slice {us[0]:6.1f}  contract {us[1]:7.1f} us ({ebytes/us[1]/1e3:6.0f} GB/s E, "
              f"{2*macs*8*(2 if ell>16 else 1)/us[1]/1e6:6.0f} TOPS)  pack {us[2]:6.1f}", flush=True)
        del w
