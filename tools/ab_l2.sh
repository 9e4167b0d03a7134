for l2 in rotate write; do
for v in base:libnimbus_cop_base.so cur:libnimbus_cop.so; do
  IFS=: read name lib <<< "$v"
  for CFG in 2 3; do
  r=$(NIMBUS_LIB=$lib timeout 120 python bench.py --config $CFG --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --l2 $l2 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), d['stages_ms_per_step_profiled'])")
  echo "$l2 cfg$CFG $name $r"
  done
done; done
FLUSH=rotate python tools/trace_tc.py 4096 2 16 1 768 768 128 2>&1 | tail -14
