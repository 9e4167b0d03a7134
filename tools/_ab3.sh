python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cop_matmul_parity or fused_r1 or same_x or kernel_variants or resident or ell64_parity or c4_full" 2>&1 | tail -2
VARS="${VARS:-}" CFGS="${CFGS:-2qkv 3 2 4}" STEPS=200 bash tools/_ab.sh
