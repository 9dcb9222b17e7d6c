timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "base_fold" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_sessions.py tests/test_gpu_golden_scale.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/breakdown.py --log2n 25 2>&1 | head -4
timeout 300 python tools/vfy_split.py 20 2>&1 | head -4
