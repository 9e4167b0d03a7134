python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -q --timeout 200 -k "host or same_x or guard" > gpurun_out/thb.log 2>&1; tail -1 gpurun_out/thb.log; grep -E '^FAILED' gpurun_out/thb.log | head
for cfg in 2qkv 2 3 2qkv; do
  timeout 300 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-graph > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);e=d['e2e'];print('$cfg', round(d['ms_per_step']*1e3,2), 'e2e', round(e['ms_per_step']*1e3,2), 'us', e['h2d_bytes_per_step'], e['d2h_bytes_per_step'], 'single', round(e['single_call']['ms_per_step']*1e3,1))" || tail -3 gpurun_out/ab.err
done
