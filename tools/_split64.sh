python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
PT="--timeout 180 --timeout-method=thread"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_rerand.py -q $PT -k "ell64 or u64 or guard or kernel_variants or rerand" > gpurun_out/ts64.log 2>&1; tail -1 gpurun_out/ts64.log; grep -E '^FAILED|Timeout' gpurun_out/ts64.log | head
NIMBUS_VARIANT=no_split python -c "from paper_2411_15707_b200 import _build; _build.build()" >/dev/null 2>&1
for r in 1 2; do for lib in "" libnimbus_cop_no_split.so; do
  if [ -n "$lib" ]; then export NIMBUS_LIB=$lib; else unset NIMBUS_LIB; fi
  for cfg in 4l64 5l64; do
    st=100; [ $cfg = 5l64 ] && st=4
    timeout 300 python bench.py --config $cfg --steps $st --warmup 2 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg', '${lib:-base}', round(d['ms_per_step'],3), 'launch', round(d['roofline']['launch_ms'],3), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done; done
