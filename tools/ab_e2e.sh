# A/B of the e2e (pipelined host-buffer) number across library builds, same box, back to back
CFG=${CFG:-2}
for rep in 1 2 3; do
for v in ${VARIANTS:-base:libnimbus_cop_base.so cur:libnimbus_cop.so}; do
  IFS=: read name lib <<< "$v"
  r=$(NIMBUS_LIB=$lib timeout 300 python bench.py --config $CFG --steps 100 --warmup 5 --no-cpu-baseline --no-stage-profile 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); e=d['e2e']; print(round(d['ms_per_step']*1000,2), round(e['ms_per_step']*1000,2), round(e['single_call']['ms_per_step']*1000,2))")
  echo "cfg$CFG $name step/e2e/single(us) $r"
done; done
