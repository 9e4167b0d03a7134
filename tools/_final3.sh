python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
bash tools/profile_round.sh r02d 4l64 5l64 > gpurun_out/profile.log 2>&1; tail -2 gpurun_out/profile.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/final_pytest.log 2>&1; tail -1 gpurun_out/final_pytest.log; grep -E '^(FAILED|ERROR)' gpurun_out/final_pytest.log | head
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc $?
