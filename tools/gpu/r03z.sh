timeout 600 python tools/verify_mem.py lenet 128 2>&1 | tail -5
timeout 600 python tools/verify_mem.py 18 2>&1 | tail -4
