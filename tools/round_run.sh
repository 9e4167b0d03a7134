#!/bin/bash
# A round-end validation run: build, GPU tests, smoke, the default bench line, ncu captures.
# PROFILE="5 5l16 ..." picks the configs to capture (default: every line of the bench).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/full_pytest.log 2>&1; tail -2 gpurun_out/full_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc $?
bash tools/profile_round.sh r02 ${PROFILE:-5 2 2qkv 3 4 4l16 5l16 4l64} > gpurun_out/profile.log 2>&1; tail -8 gpurun_out/profile.log
