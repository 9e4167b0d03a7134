python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for cfg in 2 3 2 3; do for r in 1 2; do
  NIMBUS_RES=$r timeout 300 python bench.py --config $cfg --steps 400 --warmup 10 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg', 'RES=$r', round(d['ms_per_step']*1e3,2), 'us', d['roofline']['kernel'], 'frac', round(d['roofline']['frac'],3), 'launch', round(d['roofline']['launch_ms']*1e3,2), d['clocks']['sm_mhz'])"
done; done
