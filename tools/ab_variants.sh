#!/bin/bash
# A/B timing of library builds: VARS = NIMBUS_VARIANT names (built as libnimbus_cop_<v>.so), CFGS = bench
# configs; one bench line per (config, build).  Run on the GPU box from the repo root.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in $VARS; do NIMBUS_VARIANT=$v python -c "from paper_2411_15707_b200 import _build; _build.build()"; done
for cfg in $CFGS; do
for lib in "" $VARS; do
  if [ -n "$lib" ]; then export NIMBUS_LIB=libnimbus_cop_$lib.so; else unset NIMBUS_LIB; fi
  timeout 300 python bench.py --config $cfg --steps ${STEPS:-200} --warmup 10 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg', '${lib:-base}', round(d['ms_per_step']*1e3,2), 'us', d['roofline']['kernel'], 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done; done
