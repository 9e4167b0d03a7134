python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_chain.py tests/test_gpu_graph.py -q -k "cop_matmul_parity or fused or same_x or kernel_variants or resident or random_shapes or guard or chain or graph or handles" > gpurun_out/t8.log 2>&1; tail -1 gpurun_out/t8.log; grep -E '^FAILED' gpurun_out/t8.log | head
for v in $VARS; do NIMBUS_VARIANT=$v python -c "from paper_2411_15707_b200 import _build; _build.build()" >/dev/null 2>&1; done
CFGS="3 2qkv 2 3 2qkv 2" STEPS=400 bash tools/_ab.sh
NIMBUS_TRACE=1 python -c "from paper_2411_15707_b200 import _build; _build.build()" > gpurun_out/build_trace.log 2>&1 || tail -3 gpurun_out/build_trace.log
QKV=1 FLUSH=write timeout 300 python tools/trace_tc.py 4096 2 16 1 768 768 128 2>&1 | tail -1
FLUSH=rotate timeout 300 python tools/trace_tc.py 4096 2 16 1 768 3072 128 2>&1 | tail -1
FLUSH=rotate timeout 300 python tools/trace_tc.py 4096 2 16 1 768 768 128 2>&1 | tail -1
