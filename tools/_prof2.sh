python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "packed or c5_layer or batch" > gpurun_out/tp.log 2>&1; tail -1 gpurun_out/tp.log; grep -E '^FAILED' gpurun_out/tp.log | head
timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/c5.json 2>gpurun_out/c5.err; python -c "import json;d=json.loads(open('gpurun_out/c5.json').read().strip().splitlines()[-1]);print('C5', d['ms_per_step'], d['stages_ms_per_step_profiled'], d['clocks'])"
bash tools/profile_round.sh r02b 5 5l64 2 2qkv 3 4 4l64 > gpurun_out/profile.log 2>&1; tail -8 gpurun_out/profile.log
