# k = 128 diagnostics: pure-stream floor at the QKV size, and the resident kernel's stream-only / no-epilogue variants
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_cold stream_cold.cu) || exit 1
for mb in 50 150; do echo "== stream_cold MB=$mb"; MB=$mb timeout 120 tools/stream_cold; done > gpurun_out/stream_cold.log 2>&1
cat gpurun_out/stream_cold.log
VARS="res_nomma res_noepi res_x0up res_kps1" CFGS="2qkv 3 2" STEPS=200 bash tools/_ab.sh
NIMBUS_TRACE=1 python -c "from paper_2411_15707_b200 import _build; _build.build()" > gpurun_out/build_trace.log 2>&1 || tail -3 gpurun_out/build_trace.log
for mode in rotate write; do echo "== trace C3 $mode"; FLUSH=$mode timeout 300 python tools/trace_tc.py 4096 2 16 1 768 3072 128; echo "== trace C2 $mode"; FLUSH=$mode timeout 300 python tools/trace_tc.py 4096 2 16 1 768 768 128; done > gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
