python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
NIMBUS_FUZZ_CASES=400 NIMBUS_FUZZ_SEED=9090 timeout 1800 python -m pytest tests/test_gpu_parity.py -q -k random_shapes > gpurun_out/soak.log 2>&1; tail -1 gpurun_out/soak.log; grep -E '^FAILED' gpurun_out/soak.log | head
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/full.log 2>&1; tail -1 gpurun_out/full.log; grep -E '^(FAILED|ERROR)' gpurun_out/full.log | head
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
