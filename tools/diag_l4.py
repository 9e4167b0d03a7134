"""Compare fused vs three-kernel vs oracle outputs for one shape; report where they differ."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nimbus_inputs as ni
from paper_2411_15707_b200 import nimbus as nb
from oracle import oracle as O
N, L, ell, Lo, m, n, kq = (int(x) for x in sys.argv[1:8])
res = {}
for fused in (1, 0):
    os.environ["NIMBUS_NO_FUSED"] = "0" if fused else "1"
    ctx = nb.nimbus_ctx_create(N, L, ell, Lo)
    pr = np.array(nb.nimbus_ctx_primes(ctx), np.uint32)
    sk = nb.nimbus_keygen(ctx, 5)
    W = ni.gen_W(7, m, n, ell); X = ni.gen_X(8, kq, m, ell)
    w = nb.nimbus_encrypt_weights(ctx, sk, nb.from_numpy_u32(W, "cuda"), 9)
    ws = nb.alloc_workspace(ctx, w, kq)
    cts, R = nb.alloc_outputs(ctx, w, kq, 1)
    nb.nimbus_cop_matmul(ctx, w, nb.from_numpy_u32(X, "cuda"), kq, 1, 11, cts, R, ws)
    nb.nimbus_sync(ctx)
    res[fused] = (nb.to_numpy_u32(cts), nb.to_numpy_u32(R))
    E = nb.to_numpy_u32(nb.nimbus_encw_export(w))
s = O.keygen(N, 5)
Eo = O.encrypt_rows(N, L, pr, ell, s, W, 9)
print("encw equal oracle:", (E == Eo).all())
co, Ro = O.cop_matmul(N, L, Lo, pr, ell, Eo, X, n, kq, 1, 11)
for f in (1, 0):
    c, r = res[f]
    d = c != co
    print("fused" if f else "3-kernel", "cts diff count", d.sum(), "of", d.size, "R equal", (r == Ro).all())
    if d.any():
        idx = np.argwhere(d)
        print("  first diffs (q,ct,comp,limb,J):", idx[:8].tolist())
        for ax, name in ((2, "comp"), (3, "limb")):
            print("  diffs per", name, [int(d.take(i, axis=ax).sum()) for i in range(d.shape[ax])])
