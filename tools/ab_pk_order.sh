#!/bin/bash
# A/B of the packed contraction's unit order and Enc(W) L2 policy (NIMBUS_PK_ORDER=0/1, NIMBUS_PK_EPOL=0/1/2)
# on the C5 pass: parity of the packed cases under the switches, the pass time, and the kernel's DRAM bytes
# (ncu, a few metrics: one replay pass).  COMBOS="order:epol ..."; run on the GPU box from the repo root.
mkdir -p gpurun_out
COMBOS=${COMBOS:-"0:0 1:0 1:1 1:2"}
if [ -n "${PARITY:-}" ]; then
  for c in $PARITY; do
    NIMBUS_PK_ORDER=${c%%:*} NIMBUS_PK_EPOL=${c##*:} timeout 1200 python -m pytest tests -q -m gpu -k "packed or c5_layer" > gpurun_out/order_pytest_$c.log 2>&1
    echo "parity $c: $(tail -1 gpurun_out/order_pytest_$c.log)"
  done
fi
for cfg in ${CFGS:-5}; do
for rep in 1 2; do
for c in $COMBOS; do
  NIMBUS_PK_ORDER=${c%%:*} NIMBUS_PK_EPOL=${c##*:} timeout 600 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-graph \
      > gpurun_out/order_$c.json 2> gpurun_out/order_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/order_$c.json').read().strip().splitlines()[-1]);print('C$cfg order:epol $c', round(d['ms_per_step'],3), 'ms', d['roofline']['kernel'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/order_$c.err
done
done
for c in $COMBOS; do
  NIMBUS_PK_ORDER=${c%%:*} NIMBUS_PK_EPOL=${c##*:} timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k regex:k_cop_pk -s 1 -c 1 --csv --log-file gpurun_out/order_${cfg}_dram_$c.csv \
      python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph --no-stage-profile > gpurun_out/order_ncu_$c.log 2>&1
  echo "C$cfg $c: $(grep -o '"dram__bytes_read.sum","byte","[0-9]*"\|"dram__bytes_write.sum","byte","[0-9]*"\|"gpu__time_duration.sum","ns","[0-9]*"\|"lts__t_sector_hit_rate.pct","%","[0-9.]*"' gpurun_out/order_${cfg}_dram_$c.csv | tr '\n' ' ')"
done
done
