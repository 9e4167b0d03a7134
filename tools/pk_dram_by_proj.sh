#!/bin/bash
# DRAM bytes of the packed contraction per projection type of the C5 pass (ncu, one replay pass each):
# where the pass's excess over the SURVEY 8(d) bytes comes from.  Run on the GPU box from the repo root.
mkdir -p gpurun_out
for p in ${PROJS:-Q up down}; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k regex:k_cop_pk -s 1 -c 1 --csv --log-file gpurun_out/dram_proj_$p.csv \
      python bench.py --config 5:$p --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph --no-stage-profile > gpurun_out/dram_proj_$p.log 2>&1
  echo "C5:$p (ORDER=${NIMBUS_PK_ORDER:-default}): $(grep -o '"dram__bytes_read.sum","byte","[0-9]*"\|"dram__bytes_write.sum","byte","[0-9]*"\|"gpu__time_duration.sum","ns","[0-9]*"\|"lts__t_sector_hit_rate.pct","%","[0-9.]*"' gpurun_out/dram_proj_$p.csv | tr '\n' ' ')"
done
