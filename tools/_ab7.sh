python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/t7.log 2>&1; tail -1 gpurun_out/t7.log; grep -E '^(FAILED|ERROR)' gpurun_out/t7.log | head
CFGS="3 2qkv 2" STEPS=400 bash tools/_ab.sh
NIMBUS_TRACE=1 NIMBUS_VARIANT=res_xodd python -c "from paper_2411_15707_b200 import _build; _build.build()" > gpurun_out/build_trace.log 2>&1 || tail -3 gpurun_out/build_trace.log
NIMBUS_VARIANT=res_xodd FLUSH=rotate timeout 300 python tools/trace_tc.py 4096 2 16 1 768 768 128 2>&1 | head -9
