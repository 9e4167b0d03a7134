#!/bin/bash
# Cycle accounting of the packed contraction (NIMBUS_TRACE build; tools/pk_stats.py).
NIMBUS_TRACE=1 python -c "from paper_2411_15707_b200 import _build; _build.build()" > gpurun_out/build_trace.log 2>&1 || tail -5 gpurun_out/build_trace.log
for pr in ${PROJS:-"Q,K,V,O,up,down" "up" "down"}; do echo "== $pr"; NIMBUS_PK_CL=2 timeout 600 python tools/pk_stats.py --projs $pr $ARGS 2>&1 | tail -6; done
