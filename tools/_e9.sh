python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
NIMBUS_VARIANT=pk_e9 python -c "from paper_2411_15707_b200 import _build; _build.build()" >/dev/null 2>&1
NIMBUS_LIB=libnimbus_cop_pk_e9.so timeout 300 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -k "packed" 2>&1 | tail -1
for r in 1 2 3; do for lib in "" libnimbus_cop_pk_e9.so; do
  if [ -n "$lib" ]; then export NIMBUS_LIB=$lib; else unset NIMBUS_LIB; fi
  timeout 300 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/c5.json 2>gpurun_out/c5.err
  python -c "import json;d=json.loads(open('gpurun_out/c5.json').read().strip().splitlines()[-1]);print('C5', '${lib:-base}', round(d['ms_per_step'],2), round(d['roofline']['launch_ms'],2), d['clocks']['sm_mhz'])"
done; done
