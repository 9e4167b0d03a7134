#!/bin/bash
# A/B of nimbus_cop_prefetch_next on the k = 128 configs (same box, back to back):
# block-timed step, per-step median, contraction launch (pass B events), all in us.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
python -m pytest tests/test_gpu_parity.py -q -k "prefetch_next" 2>&1 | tail -1
for rep in 1 2 3; do
for cfg in ${CFGS:-3 2 2qkv}; do
for pf in ${PFS:-0 1}; do
  r=$(timeout 200 python bench.py --config $cfg --steps ${STEPS:-400} --warmup 10 --no-cpu-baseline --no-e2e --no-graph --prefetch-next $pf 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), round(d['step_ms_dist']['median']*1000,2), round(d['roofline']['launch_ms']*1000,2), d['clocks']['sm_mhz'])")
  echo "cfg$cfg prefetch_next=$pf block/per-step/launch(us) clk: $r"
done; done; done
