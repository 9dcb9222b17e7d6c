timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "lane16" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/vfy_split.py 20 2>&1 | head -16 | tail -9
