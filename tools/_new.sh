python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rerand.py -q -x -k "u64 or rerand or streamed or ell64_full or packed or same_x" > gpurun_out/new_pytest.log 2>&1; tail -15 gpurun_out/new_pytest.log
