timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "mul16 or lane16" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py tests/test_gpu_sessions.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/vfy_split.py 20 2>&1 | head -9
timeout 900 python tools/verify_mem.py lenet 256 2>&1 | tail -3
