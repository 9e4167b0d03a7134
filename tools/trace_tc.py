"""Timeline of the tcgen05 contraction kernel from the debug trace build
(NIMBUS_TRACE=1 python paper_2411_15707_b200/_build.py): per-CTA setup,
PDL wait, per-tile MMA and epilogue intervals (globaltimer ns)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import nimbus_inputs as ni
from paper_2411_15707_b200 import nimbus as nb

_var = os.environ.get("NIMBUS_VARIANT", "")
nb.LIB_PATH = os.path.join(os.path.dirname(nb.LIB_PATH), "libnimbus_cop_trace" + (f"_{_var}" if _var else "") + ".so")
lib = nb.lib()
cfg = ni.get = None
N, L, ell, Lo, m, n, k = (int(x) for x in sys.argv[1:8])
ctx = nb.nimbus_ctx_create(N, L, ell, Lo)
sk = nb.nimbus_keygen(ctx, 1)
w = nb.nimbus_encrypt_weights(ctx, sk, nb.from_numpy_u32(ni.gen_W(1, m, n, ell), "cuda"), 1)
X = nb.from_numpy_u32(ni.gen_X(2, k, m, ell), "cuda")
ws = nb.alloc_workspace(ctx, w, k)
cts, R = nb.alloc_outputs(ctx, w, k, 1)
tr = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
rflush = torch.ones(64 << 20, dtype=torch.int32, device="cuda")   # 256 MB read: leaves L2 clean
MODE = os.environ.get("FLUSH", "write")
for _ in range(3):
    nb.nimbus_cop_matmul(ctx, w, X, k, 1, 3, cts, R, ws)
others = []
if MODE == "rotate":   # as bench --l2 rotate: other copies' inputs fill the L2 (clean lines)
    Wd = nb.from_numpy_u32(ni.gen_W(1, m, n, ell), "cuda")
    others = [(nb.nimbus_encrypt_weights(ctx, sk, Wd, 1), X.clone()) for _ in range(7)]
    flush.zero_()
    for wo, Xo in others:
        nb.nimbus_cop_matmul(ctx, wo, Xo, k, 1, 3, cts, R, ws)
lib.nimbus_trace_set(ctypes.c_void_p(tr.data_ptr()))
trp = torch.tensor([2**62, 2**62, 0, 0], dtype=torch.int64, device="cuda")
lib.nimbus_trace_pack_set(ctypes.c_void_p(trp.data_ptr()))
if MODE in ("write", "writeread"):
    flush.zero_()
if MODE == "writeread":
    rflush.sum()
torch.cuda.synchronize()
if os.environ.get("QKV") == "1":
    # Q, K, V sharing X: one batch call (one resident-X launch over the three Enc(W)s)
    ws3 = [(nb.nimbus_encrypt_weights(ctx, sk, nb.from_numpy_u32(ni.gen_W(5 + i, m, n, ell), "cuda"), 5 + i),)
           for i in range(3)]
    outs = [nb.alloc_outputs(ctx, wq[0], k, 1) for wq in ws3]
    jobs = [dict(encw=wq[0], X=X, k_per_query=k, n_queries=1, mask_seed=3, cts=o[0], R=o[1])
            for wq, o in zip(ws3, outs)]
    wsb = torch.empty(nb.nimbus_cop_workspace_size_batch(ctx, jobs), dtype=torch.uint8, device="cuda")
    nb.nimbus_cop_matmul_batch(ctx, jobs, wsb)
    torch.cuda.synchronize()
    tr.zero_()
    flush.zero_()
    torch.cuda.synchronize()
    nb.nimbus_cop_matmul_batch(ctx, jobs, wsb)
else:
    nb.nimbus_cop_matmul(ctx, w, X, k, 1, 3, cts, R, ws)
torch.cuda.synchronize()
lib.nimbus_trace_set(ctypes.c_void_p(0))
lib.nimbus_trace_pack_set(ctypes.c_void_p(0))
t = tr.cpu().numpy().reshape(148, 64).astype(np.int64)
t0 = t[:, 0][t[:, 0] > 0].min()
us = lambda x: (x - t0) / 1e3 if x > 0 else float("nan")
print(f"N={N} L={L} ell={ell} m={m} n={n} k={k}")
ends = []
for c in (0, 1, 2, 50, 100, 147):
    row = t[c]
    s = f"cta {c:3d}: start {us(row[0]):6.2f} setup {us(row[1]):6.2f} pdl {us(row[2]):6.2f} end {us(row[3]):6.2f} |"
    for ti in range(15):
        if row[4 + 4 * ti] == 0:
            break
        s += f" t{ti}: mma {us(row[4+4*ti]):.1f}-{us(row[5+4*ti]):.1f} epi {us(row[6+4*ti]):.1f}-{us(row[7+4*ti]):.1f} |"
    print(s)
if (t[:, 61] > 0).any():
    for c in (0, 1, 100, 147):
        row = t[c]
        print(f"cta {c}: 3rd E copy issued {us(row[63]):.2f} first E landed {us(row[60]):.2f} "
              f"X: past PDL wait {us(row[61]):.2f} rows written {us(row[62]):.2f}")
for c in (0, 100):
    row = t[c]
    print(f"cta {c} tile1 producer B issue:", " ".join(f"{us(row[52+i]):.2f}" for i in range(8) if row[52+i] > 0))
    print(f"cta {c} tile1 MMA full ready :", " ".join(f"{us(row[40+i]):.2f}" for i in range(8) if row[40+i] > 0))
e = np.array([us(x) for x in t[:, 3] if x > 0])
print(f"CTA end: min {e.min():.2f} median {np.median(e):.2f} max {e.max():.2f} us")
st = np.array([us(x) for x in t[:, 0] if x > 0])
print(f"CTA start: min {st.min():.2f} max {st.max():.2f}")
tp = trp.cpu().numpy().astype(np.int64)
print(f"pack: first block start {us(tp[0]):.2f}  first past PDL wait {us(tp[1]):.2f}  last past wait {us(tp[2]):.2f}  "
      f"last block end {us(tp[3]):.2f} us (contraction CTAs end max {e.max():.2f})")
# aggregate over CTAs: first-tile MMA end, later tiles' MMA spans, the final epilogue (the tail)
t0_end, spans, tails = [], [], []
for c in range(148):
    row = t[c]
    if row[0] == 0 or row[4] == 0:
        continue
    nt = 0
    while nt < 15 and row[4 + 4 * nt] > 0:
        nt += 1
    t0_end.append(us(row[5]))
    for ti in range(1, nt):
        spans.append((row[5 + 4 * ti] - row[5 + 4 * (ti - 1)]) / 1e3)
    tails.append((row[7 + 4 * (nt - 1)] - row[5 + 4 * (nt - 1)]) / 1e3)
if t0_end:
    print(f"first tile MMA end: median {np.median(t0_end):.2f} max {np.max(t0_end):.2f} us; later tiles (MMA end to "
          f"MMA end): median {np.median(spans) if spans else float('nan'):.2f} us; final epilogue after the last MMA: "
          f"median {np.median(tails):.2f} max {np.max(tails):.2f} us")
