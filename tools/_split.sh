python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
PT="--timeout 120 --timeout-method=thread"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -q $PT -k "cop_matmul_parity or c4_full or kernel_variants or guard or accumulate or batch or host" > gpurun_out/ts.log 2>&1; tail -1 gpurun_out/ts.log; grep -E '^FAILED|Timeout' gpurun_out/ts.log | head
NIMBUS_FUZZ_CASES=300 NIMBUS_FUZZ_SEED=31337 timeout 400 python -m pytest tests/test_gpu_parity.py -q $PT -k random_shapes 2>&1 | tail -1


