python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in $VARS; do NIMBUS_VARIANT=$v python -c "from paper_2411_15707_b200 import _build; _build.build()" > /dev/null 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "encrypt or c4_full or smoke" 2>&1 | tail -2
for c in 2 4 5; do
  for lib in "" $VARS; do
    if [ -n "$lib" ]; then export NIMBUS_LIB=libnimbus_cop_$lib.so; else unset NIMBUS_LIB; fi
    timeout 300 python tools/bench_setup.py --config $c 2>&1 | tail -1
  done
  unset NIMBUS_LIB
  NIMBUS_ENC_TWOPASS=1 timeout 300 python tools/bench_setup.py --config $c 2>&1 | tail -1
done
