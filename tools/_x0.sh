python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
NIMBUS_VARIANT=res_x0up python -c "from paper_2411_15707_b200 import _build; _build.build()"
NIMBUS_LIB=libnimbus_cop_res_x0up.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cop_matmul_parity or fused_r1 or same_x or random_shapes or kernel_variants" 2>&1 | tail -2
VARS="res_x0up" CFGS="2 2qkv 3" bash tools/_ab.sh
