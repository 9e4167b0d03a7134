python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for cfg in 2 2qkv 2 2qkv; do for v in 1 2 4; do
  NIMBUS_PACK_V=$v timeout 300 python bench.py --config $cfg --steps 400 --warmup 10 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg', 'V=$v', round(d['ms_per_step']*1e3,2), 'us', 'pack', round(d['stages_ms_per_step_profiled']['pack_moddown_mask']*1e3,2), d['clocks']['sm_mhz'])"
done; done
