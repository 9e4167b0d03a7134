#!/usr/bin/env python
"""Markdown table of a bench.py line (default: profiles/round2_bench/bench_default.json) for DESIGN.md / README.md."""
import json
import sys

d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "profiles/round2_bench/bench_default.json"))


def t(ms):
    return f"{ms:.1f} ms" if ms >= 5 else f"{ms * 1e3:.1f} µs"


print("| config | step | value (modMAC/s) | contraction kernel (per launch) | roofline, per launch | whole step | vs measured i8 rate | e2e / step | SM clock |")
print("|---|---|---|---|---|---|---|---|---|")
for name, x in [(d["config"]["config"], d)] + list(d.get("per_config", {}).items()):
    r, f, s = x["roofline"], x.get("roofline_i8_floor"), x.get("roofline_step")
    fl = f"{f['frac']:.3f}" if f and r["bound"] == "tensor" else "—"
    st = f"{s['frac']:.3f}" if s else "—"
    e = x.get("e2e", {}).get("ms_per_step")
    print(f"| {name} | {t(x['ms_per_step'])} | {x['value']:.2e} | `{r['kernel']}` ({t(r['launch_ms'])} × {r['launches_per_step']:.0f}) | "
          f"{r['bound']} {r['frac']:.3f} | {st} | {fl} | {t(e) if e else '—'} | {x['clocks']['sm_mhz']:.0f} MHz "
          f"{'(' + ','.join(x['clocks']['reasons']) + ')' if x['clocks']['reasons'] else ''} |")
