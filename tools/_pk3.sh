python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "packed or c5_layer" > gpurun_out/pk_pytest.log 2>&1; tail -3 gpurun_out/pk_pytest.log
for v in 0 1; do
  NIMBUS_NO_PACKED=$v timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab_C5_$v.json 2> gpurun_out/ab_C5_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_C5_$v.json').read().strip().splitlines()[-1]);print('NO_PACKED=$v', d['ms_per_step'], d['stages_ms_per_step_profiled'], d['clocks'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cop_pk -c 1 -o gpurun_out/pk_C5_prof -f python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph --no-stage-profile > gpurun_out/pk_ncu.log 2>&1
echo ncu rc $?
