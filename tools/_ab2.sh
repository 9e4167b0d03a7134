timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "packed or c5_layer" 2>&1 | tail -2
bash tools/_ab.sh
