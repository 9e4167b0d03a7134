python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "test_random_shapes_parity and 128-3-24-2-86-12-45-1" > gpurun_out/t2a.log 2>&1; tail -1 gpurun_out/t2a.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "random_shapes" > gpurun_out/t2b.log 2>&1; tail -1 gpurun_out/t2b.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "fused or random_shapes" > gpurun_out/t2c.log 2>&1; tail -1 gpurun_out/t2c.log; grep -E '^FAILED' gpurun_out/t2c.log
git stash -q 2>/dev/null; echo no-git
