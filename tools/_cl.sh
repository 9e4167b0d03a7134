python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "packed or c5_layer" 2>&1 | tail -2
for sub in ${SUBS:-5 "5:Q,K,V,O" "5:up" "5:down"}; do
  NIMBUS_PK_CL=2 timeout 300 python bench.py --config "$sub" --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$sub', round(d['ms_per_step'],3), d['roofline']['kernel'], 'i8floor', round(d['roofline_i8_floor']['frac'],3), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" || tail -3 gpurun_out/ab.err
done
[ -n "$STATS" ] && bash tools/_stats.sh
true
