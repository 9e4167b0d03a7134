(cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_cold stream_cold.cu) || exit 1
for h in 0 1000 2000; do HOLD_NS=$h MB=150 timeout 120 tools/stream_cold | grep hold; done
