B="python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
for rep in 1 2; do for cfg in 2 3; do for r in 1 2; do
  v=$(NIMBUS_RES=$r timeout 120 $B --config $cfg 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), d['stages_ms_per_step_profiled']['contraction']*1000, d['roofline']['frac'])")
  echo "cfg$cfg res$r $v"
done; done; done
