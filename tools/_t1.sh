python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_chain.py tests/test_gpu_graph.py -q -k "cop_matmul_parity or fused or same_x or kernel_variants or resident or random_shapes or guard or chain or graph" > gpurun_out/t1.log 2>&1; tail -2 gpurun_out/t1.log; grep -E '^(FAILED|ERROR)' gpurun_out/t1.log | head
NIMBUS_VARIANT=res_xhalf python -c "from paper_2411_15707_b200 import _build; _build.build()" >/dev/null 2>&1
VARS="res_xhalf" CFGS="3 2qkv 2" STEPS=400 bash tools/_ab.sh
