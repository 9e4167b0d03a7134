python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
K="cop_matmul_parity or fused or same_x or kernel_variants or resident or random_shapes"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "$K" > gpurun_out/t3a.log 2>&1; tail -1 gpurun_out/t3a.log; grep -E '^FAILED' gpurun_out/t3a.log
(cd headcopy && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/buildh.log 2>&1 && timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "$K" > ../gpurun_out/t3b.log 2>&1; tail -1 ../gpurun_out/t3b.log; grep -E '^FAILED' ../gpurun_out/t3b.log)
