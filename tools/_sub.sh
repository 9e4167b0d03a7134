# per-projection subsets of C5: time + DRAM bytes of the packed contraction
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for sub in ${SUBS:-"5:Q,K,V,O" "5:up" "5:down"}; do
  timeout 300 python bench.py --config "$sub" --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$sub', round(d['ms_per_step'],3), d['roofline']['kernel'], 'i8floor', round(d['roofline_i8_floor']['frac'],3), 'alg GB', round(d['roofline_other']['achieved']*d['roofline']['launch_ms']/1e3,2), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:k_cop_pk -c 1 --csv python bench.py --config "$sub" --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph 2>/dev/null | grep -E '"(dram|gpu__|lts)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
