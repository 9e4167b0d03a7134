"""Run tools/mma_bench (tcgen05 kind::i8, M = 128, both operands in shared memory) on the GPU
box and write profiles/mma_bench.json: the N = 256 burst rate (one ~1 ms launch) and the
sustained rate (back-to-back launches for ~4 s, under the board power limit), with the SM
clock sampled during the sustained run.  bench.py reads `tops_n256` (the sustained figure:
the C5 pass is a ~100 ms tensor-bound kernel) as its measured kind::i8 floor."""
import json
import os
import subprocess
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

clk = bench.ClockSampler(0)
clk.start()
out = subprocess.run([os.path.join(ROOT, "tools", "mma_bench"), "json"], capture_output=True, text=True).stdout
c = clk.stop()
rows = [json.loads(l[5:]) for l in out.splitlines() if l.startswith("JSON ")]
burst = {r["n"]: r for r in rows if "n" in r}
sus = [r["sustained_tops_n256"] for r in rows if "sustained_tops_n256" in r]
res = {"src": "tools/mma_bench.cu on B200 (tools/mma_bench_json.py)",
       "burst": burst, "sustained_tops_n256": sus[0] if sus else None,
       "tops_n256": sus[0] if sus else burst.get(256, {}).get("tops"),
       "clocks_during_sustained": c, "raw": out}
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "profiles", "mma_bench.json"), "w"), indent=1)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)       # travels back from the GPU box
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "mma_bench.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "raw"}))
