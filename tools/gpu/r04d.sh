timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "matmul or rows_times or tc or table" 2>&1 | tail -2
timeout 600 python tools/breakdown.py --log2n 25 2>&1 | head -12
