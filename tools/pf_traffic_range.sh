#!/bin/bash
# DRAM bytes of K chained steps as they really run (PDL overlap, no serialisation, no cache flush):
# ncu range replay over the block-timed pass of bench.py, one pass.  Per step = total / K.
mkdir -p gpurun_out
K=${K:-40}
for c in ${CFGS:-3 2}; do for pf in 0 1; do
  timeout 600 ncu --replay-mode range --cache-control none --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
      --csv --log-file gpurun_out/pf_range_C${c}_pf$pf.csv \
      python bench.py --config $c --steps $K --warmup 5 --prefetch-next $pf --profiler-range --no-cpu-baseline --no-e2e --no-graph --no-stage-profile > gpurun_out/pf_range_C${c}_pf$pf.log 2>&1
  echo "C$c prefetch_next=$pf, $K steps in one range: $(grep -o '"dram__bytes_read.sum","[a-zA-Z]*","[0-9.,]*"\|"dram__bytes_write.sum","[a-zA-Z]*","[0-9.,]*"\|"lts__t_sector_hit_rate.pct","%","[0-9.]*"' gpurun_out/pf_range_C${c}_pf$pf.csv | tr '\n' ' ')"
done; done
