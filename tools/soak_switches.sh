#!/bin/bash
# Random-shape soak of every kernel-selection switch: 300 seeded shapes plus
# the packed and same-X group cases per switch, each compared bit-exactly with the oracle.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
PT="--timeout 300 --timeout-method=thread"
for env in "NIMBUS_PACK_V=1" "NIMBUS_PACK_V=4" "NIMBUS_RES=2" "NIMBUS_NO_FUSE=1" "NIMBUS_TRANSPOSED=1" "NIMBUS_NO_GROUP=1" "NIMBUS_PK_CL=1" "NIMBUS_PK_CL=4" "NIMBUS_NO_PACKED=1"; do
  r=$(env $env NIMBUS_FUZZ_CASES=300 NIMBUS_FUZZ_SEED=5150 timeout 600 python -m pytest tests/test_gpu_parity.py -q $PT -k "random_shapes or packed or same_x" 2>&1 | tail -1)
  echo "$env: $r"
done
