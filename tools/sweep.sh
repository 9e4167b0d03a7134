# Full bench sweep of every config line (one box, back to back) -> gpurun_out/sweep_<cfg>.json
for c in ${CONFIGS:-1 2 3 4 4l16 4l64}; do
  timeout 600 python bench.py --config $c > gpurun_out/sweep_$c.json 2> gpurun_out/sweep_$c.err || echo "config $c failed"
done
for c in ${CONFIGS5:-5 5l16 5l64}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/sweep_$c.json 2> gpurun_out/sweep_$c.err || echo "config $c failed"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/sweep_ref2.json 2> gpurun_out/sweep_ref2.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
