python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "packed or c5_layer" > gpurun_out/pk_pytest.log 2>&1; tail -30 gpurun_out/pk_pytest.log
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/pk_C5.json 2> gpurun_out/pk_C5.err; tail -c 1500 gpurun_out/pk_C5.json; tail -5 gpurun_out/pk_C5.err
