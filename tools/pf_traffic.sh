#!/bin/bash
# DRAM bytes per resident-X contraction launch in steady state, with and without nimbus_cop_prefetch_next:
# one ncu pass per launch (no replay), caches NOT flushed between launches (--cache-control none), so a
# launch's first tiles can hit what the launch before it prefetched.  The --set full captures flush the
# caches before every replay and therefore charge a launch with its own cold first tiles AND its prefetch.
mkdir -p gpurun_out
for c in ${CFGS:-3 2}; do for pf in 0 1; do
  timeout 600 ncu --cache-control none --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
      -k regex:k_cop_tc_res -s 16 -c 24 --csv --log-file gpurun_out/pf_traffic_C${c}_pf$pf.csv \
      python bench.py --config $c --steps 20 --warmup 5 --prefetch-next $pf --no-cpu-baseline --no-e2e --no-graph --no-stage-profile > gpurun_out/pf_traffic_C${c}_pf$pf.log 2>&1
  python - <<P
import csv, statistics
rows = [r for r in csv.reader(l for l in open("gpurun_out/pf_traffic_C${c}_pf$pf.csv") if l.startswith('"'))]
h = rows[0]; rows = rows[1:]
mi, vi = h.index("Metric Name"), h.index("Metric Value")
agg = {}
for r in rows:
    agg.setdefault(r[mi], []).append(float(r[vi].replace(",", "")))
print("C$c prefetch_next=$pf launches", len(agg.get("dram__bytes_read.sum", [])),
      {k: round(statistics.median(v) / (1e6 if "bytes" in k else 1e3 if "duration" in k else 1), 2) for k, v in agg.items()},
      "(median per launch: MB, us, %)")
P
done; done
