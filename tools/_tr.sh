python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
NIMBUS_TRACE=1 python -c "from paper_2411_15707_b200 import _build; _build.build()" > gpurun_out/build_trace.log 2>&1 || tail -3 gpurun_out/build_trace.log
QKV=1 FLUSH=write timeout 300 python tools/trace_tc.py 4096 2 16 1 768 768 128 2>&1 | tail -12
FLUSH=rotate timeout 300 python tools/trace_tc.py 4096 2 16 1 768 3072 128 2>&1 | tail -3
