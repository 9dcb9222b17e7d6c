timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_ppml.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/verify_mem.py lenet 128 2>&1 | tail -4
timeout 600 python tools/ppml_breakdown.py lenet 128 check 2>&1 | head -8
