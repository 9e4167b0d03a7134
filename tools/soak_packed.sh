#!/bin/bash
# Random-shape soak of the NIMBUS_FLAG_LARGE_K layout (packed contraction at S_x = 2 / 4 where it applies,
# transposed row-wise kernel otherwise), each shape compared bit-exactly with the oracle: the default
# build, the CTA-pair form and the old unit order.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
PT="--timeout 300 --timeout-method=thread"
for env in "NIMBUS_FUZZ_LK_CASES=${CASES:-400}" "NIMBUS_PK_PAIR=1 NIMBUS_FUZZ_LK_CASES=${CASES2:-200}" "NIMBUS_PK_ORDER=0 NIMBUS_FUZZ_LK_CASES=${CASES2:-200}"; do
  r=$(env $env NIMBUS_FUZZ_LK_SEED=${SEED:-777} timeout 1500 python -m pytest tests/test_gpu_parity.py -q $PT -k "large_k_parity" 2>&1 | tail -3 | tr '\n' ' ')
  echo "$env: $r"
done
