#!/bin/bash
# Usage (on the GPU box): tools/ncu_run.sh <tag> <kernel-regex> <bench args...>
# 1) plain run (must exit 0), 2) launch list, 3) one --set full capture of the named kernel.
tag=$1; kern=$2; shift 2
python bench.py "$@" --no-cpu-baseline --no-e2e --no-graph > gpurun_out/${tag}_plain.json 2> gpurun_out/${tag}_plain.err || { echo "plain run failed"; tail gpurun_out/${tag}_plain.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py "$@" --no-cpu-baseline --no-e2e --no-graph > gpurun_out/${tag}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${kern} -s 3 -c 1 -o gpurun_out/${tag}_prof -f \
    python bench.py "$@" --no-cpu-baseline --no-e2e --no-graph > gpurun_out/${tag}_ncu2.log 2>&1
echo "ncu done $?"
