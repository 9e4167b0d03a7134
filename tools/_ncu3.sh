python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
args="--config ${CFG:-3} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-stage-profile"
timeout 300 python bench.py $args > gpurun_out/plain.json 2> gpurun_out/plain.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cop -s 2 -c 1 \
      -o gpurun_out/${TAG:-C3}_prof -f python bench.py $args > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
