timeout 600 python tools/dots_mem.py 128 2>&1 | tail -80
