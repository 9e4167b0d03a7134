python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "feeds_next" > gpurun_out/t12a.log 2>&1; tail -1 gpurun_out/t12a.log; grep -E '^(FAILED|E  )' gpurun_out/t12a.log | head
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/t12.log 2>&1; tail -1 gpurun_out/t12.log; grep -E '^FAILED' gpurun_out/t12.log | head
CFGS="2 2qkv 3 4 2 2qkv 3 4" STEPS=300 bash tools/_ab.sh
