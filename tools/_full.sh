python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/full_pytest.log 2>&1; tail -3 gpurun_out/full_pytest.log
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o mma_bench mma_bench.cu) && timeout 300 python tools/mma_bench_json.py > gpurun_out/mma.log 2>&1; tail -2 gpurun_out/mma.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc $?; tail -3 gpurun_out/bench_default.err
