python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "packed or c5_layer or batch or kernel_variants" > gpurun_out/tp4.log 2>&1; tail -1 gpurun_out/tp4.log; grep -E '^FAILED' gpurun_out/tp4.log | head
NIMBUS_VARIANT=pk_nostagger python -c "from paper_2411_15707_b200 import _build; _build.build()" >/dev/null 2>&1
for lib in "" libnimbus_cop_pk_nostagger.so "" libnimbus_cop_pk_nostagger.so; do
  if [ -n "$lib" ]; then export NIMBUS_LIB=$lib; else unset NIMBUS_LIB; fi
  timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-stage-profile > gpurun_out/c5.json 2>gpurun_out/c5.err
  python -c "import json;d=json.loads(open('gpurun_out/c5.json').read().strip().splitlines()[-1]);print('C5', '${lib:-base}', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
done
unset NIMBUS_LIB
args="--config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph --no-stage-profile"
for lib in "" libnimbus_cop_pk_nostagger.so; do
  if [ -n "$lib" ]; then export NIMBUS_LIB=$lib; else unset NIMBUS_LIB; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_cop_pk -c 2 --csv python bench.py $args 2>/dev/null | grep -E 'dram__bytes|gpu__time|hit_rate' | tail -4 | sed "s/^/${lib:-base}: /"
done
