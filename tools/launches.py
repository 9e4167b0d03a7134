"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        agg.setdefault(r[ki][:70], []).append(float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1))
    print(path)
    for k, v in agg.items():
        print(f"  {k:70s} n={len(v):4d} mean={sum(v)/len(v):9.2f} us  min={min(v):9.2f}")
