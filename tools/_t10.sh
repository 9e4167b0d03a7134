python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "same_x or handles" > gpurun_out/t10.log 2>&1; tail -1 gpurun_out/t10.log; grep -E '^FAILED' gpurun_out/t10.log | head
bash tools/_stats.sh
