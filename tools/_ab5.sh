python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_chain.py tests/test_gpu_graph.py -x -q -k "cop_matmul_parity or fused or same_x or kernel_variants or resident or random_shapes or guard or chain or graph" 2>&1 | tail -2
for v in $VARS; do NIMBUS_VARIANT=$v python -c "from paper_2411_15707_b200 import _build; _build.build()" >/dev/null 2>&1; done
for v in $VARS; do NIMBUS_LIB=libnimbus_cop_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cop_matmul_parity or fused or same_x" 2>&1 | tail -1; done
VARS="${VARS:-}" CFGS="${CFGS:-3 2qkv 2 3 2qkv 2}" STEPS=400 bash tools/_ab.sh
