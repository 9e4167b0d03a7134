python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_rerand.py -q > gpurun_out/t11.log 2>&1; tail -1 gpurun_out/t11.log; grep -E '^FAILED' gpurun_out/t11.log | head
CFGS="2 2qkv 4 1 2 2qkv 4 1" STEPS=300 bash tools/_ab.sh
