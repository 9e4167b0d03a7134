python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 200 -k "packed or c5_layer" 2>&1 | tail -1
for r in 1 2; do for tau in 1100 0 600 2000; do
  NIMBUS_PK_TAU=$tau timeout 300 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-stage-profile > gpurun_out/c5.json 2>gpurun_out/c5.err
  python -c "import json;d=json.loads(open('gpurun_out/c5.json').read().strip().splitlines()[-1]);print('C5 tau=$tau', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
done; done
args="--config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph --no-stage-profile"
for tau in 1100 0; do
  NIMBUS_PK_TAU=$tau timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_cop_pk -c 1 --csv python bench.py $args 2>/dev/null | grep -E 'dram__bytes|gpu__time|hit_rate' | awk -F'","' '{print $(NF-2), $NF}' | sed "s/^/tau=$tau: /"
done
