mkdir -p gpurun_out
timeout 300 python tools/breakdown.py --log2n 24 --d 64 > gpurun_out/r02l_bd_mulv24.txt 2>&1
timeout 300 python tools/breakdown.py --prog relu --log2n 16 > gpurun_out/r02l_bd_relu16.txt 2>&1
