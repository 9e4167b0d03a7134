python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "packed or c5_layer" 2>&1 | tail -2
for cl in 2; do
  NIMBUS_PK_CL=$cl timeout 300 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('CL=$cl', round(d['ms_per_step'],3), d['roofline']['kernel'], round(d['stages_ms_per_step_profiled']['contraction'],3), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" || tail -3 gpurun_out/ab.err
done
NIMBUS_TRACE=1 python -c "from paper_2411_15707_b200 import _build; _build.build()" > gpurun_out/build_trace.log 2>&1 || tail -5 gpurun_out/build_trace.log
NIMBUS_PK_CL=2 timeout 600 python tools/pk_stats.py 2>&1 | tail -4
