#!/bin/bash
# Capture the round's profiles on the GPU box: for each config, the launch list of the
# bench command and one `ncu --set full` capture of its contraction kernel, summarised
# into profiles/ncu_<config>.json (bench.py's roofline `traffic` reads it).
# Usage: tools/profile_round.sh <round-tag> <config> [<config> ...]   (e.g. r02 5 2 3 4 4l64)
set -u
tag=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  case $c in 5|5l64|5l16) args="--config $c --steps 1 --warmup 1";; *) args="--config $c --steps 5 --warmup 3";; esac
  name=C$c
  common="--no-cpu-baseline --no-e2e --no-graph"
  timeout 900 python bench.py $args $common --no-stage-profile > gpurun_out/${name}_plain.json 2> gpurun_out/${name}_plain.err \
    || { echo "plain run failed for $c"; tail -3 gpurun_out/${name}_plain.err; continue; }
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
      --log-file gpurun_out/${name}_launches.csv python bench.py $args $common --no-stage-profile > gpurun_out/${name}_ncu1.log 2>&1
  timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_cop -s 2 -c 1 \
      -o gpurun_out/${name}_prof -f python bench.py $args $common --no-stage-profile > gpurun_out/${name}_ncu2.log 2>&1
  echo "profiled $c"
done
