# Per-kernel durations with L2 state preserved between kernels (ncu --cache-control none):
# closer to the in-chain behaviour than the default cold-cache launch list.
for c in "$@"; do
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 200 --csv \
      --log-file gpurun_out/C${c}_launches_warm.csv \
      python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-stage-profile > gpurun_out/C${c}_ncuw.log 2>&1
  python tools/launches.py gpurun_out/C${c}_launches_warm.csv | grep -v "FillFunctor\|keygen\|encrypt\|tile_encw"
done
