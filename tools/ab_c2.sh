# A/B of bench step time across experiment builds / env switches (same box, back to back)
# VARIANTS="name:libfile[:ENV=VAL] ..."
CFG=${CFG:-2}
B="python bench.py --config $CFG --steps 300 --warmup 10 --no-cpu-baseline --no-e2e --no-graph --no-stage-profile"
for rep in 1 2; do
for v in ${VARIANTS:-base:libnimbus_cop_base.so cur:libnimbus_cop.so}; do
  IFS=: read name lib envs <<< "$v"
  r=$(env NIMBUS_LIB=$lib $envs timeout 120 $B 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2), round(d['step_ms_dist']['median']*1000,2))")
  echo "cfg$CFG $name block/per-step(us) $r"
done; done
