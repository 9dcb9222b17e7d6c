timeout 900 python -m pytest tests/test_gpu_sessions.py -x -q -p no:cacheprovider -k lane16 2>&1 | tail -15
timeout 600 python tools/verify_mem.py lenet 128 2>&1 | tail -3
timeout 600 python tools/ppml_breakdown.py lenet 128 check 2>&1 | head -3
