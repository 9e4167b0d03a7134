python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
NIMBUS_PK_CL=4 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "packed or c5_layer" 2>&1 | tail -2
for cl in 2 4; do
for sub in 5 "5:Q,K,V,O" "5:up" "5:down"; do
  NIMBUS_PK_CL=$cl timeout 300 python bench.py --config "$sub" --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('CL=$cl', '$sub', round(d['ms_per_step'],3), d['roofline']['kernel'], 'i8floor', round(d['roofline_i8_floor']['frac'],3), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))" || tail -3 gpurun_out/ab.err
done; done
for cl in 2 4; do
  NIMBUS_PK_CL=$cl timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:k_cop_pk -c 1 --csv python bench.py --config 5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph 2>/dev/null | grep -E '"(dram|lts)' | awk -F'","' -v cl=$cl '{print "CL=" cl, $(NF-2), $(NF-1), $NF}'
done
