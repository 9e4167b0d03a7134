NIMBUS_TRACE=1 python -c "from paper_2411_15707_b200 import _build; _build.build()" > gpurun_out/build_trace.log 2>&1 || tail -5 gpurun_out/build_trace.log
for cl in 1 2; do NIMBUS_PK_CL=$cl timeout 600 python tools/pk_stats.py $ARGS 2>&1 | tail -4; done
