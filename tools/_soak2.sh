python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
PT="--timeout 300 --timeout-method=thread"
NIMBUS_FUZZ_CASES=2000 NIMBUS_FUZZ_SEED=4242 timeout 1200 python -m pytest tests/test_gpu_parity.py -q $PT -k random_shapes > gpurun_out/soak2.log 2>&1; tail -1 gpurun_out/soak2.log; grep -E '^FAILED' gpurun_out/soak2.log | head -5
NIMBUS_CLUSTER=2 NIMBUS_FUZZ_CASES=500 NIMBUS_FUZZ_SEED=777 timeout 600 python -m pytest tests/test_gpu_parity.py -q $PT -k random_shapes 2>&1 | tail -1
NIMBUS_NO_RESIDENT=1 NIMBUS_FUZZ_CASES=500 NIMBUS_FUZZ_SEED=778 timeout 600 python -m pytest tests/test_gpu_parity.py -q $PT -k random_shapes 2>&1 | tail -1
