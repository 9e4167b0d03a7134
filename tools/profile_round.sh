#!/bin/bash
# Capture the round's profiles on the GPU box: for each config, the launch list
# of the bench command and one --set full capture of the contraction kernel.
# Usage: tools/profile_round.sh <config> [<config> ...]   (e.g. 2 4)
set -u
for c in "$@"; do
  case $c in 5) args="--config 5 --steps 2 --warmup 1";; *) args="--config $c --steps 5 --warmup 3";; esac
  tag=C$c
  python bench.py $args --no-cpu-baseline --no-e2e --no-stage-profile --no-graph > gpurun_out/${tag}_plain.json 2> gpurun_out/${tag}_plain.err || { echo "plain run failed for $c"; tail -3 gpurun_out/${tag}_plain.err; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
      python bench.py $args --no-cpu-baseline --no-e2e --no-stage-profile --no-graph > gpurun_out/${tag}_ncu1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_cop_tc -s 2 -c 1 -o gpurun_out/${tag}_prof -f \
      python bench.py $args --no-cpu-baseline --no-e2e --no-stage-profile --no-graph > gpurun_out/${tag}_ncu2.log 2>&1
  echo "profiled $c"
done
