mkdir -p gpurun_out
timeout 600 python tools/verify_mem.py 18 > gpurun_out/r02n_vmem.txt 2>&1
