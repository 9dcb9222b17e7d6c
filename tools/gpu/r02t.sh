mkdir -p gpurun_out
timeout 300 python tools/breakdown.py --prog mulv --log2n 24 --d 64 > gpurun_out/r02t_bd_mulv24.txt 2>&1
for b in 128 192 256; do timeout 600 python tools/mem_probe.py lenet $b; done > gpurun_out/r02t_mem_lenet.txt 2>&1
cat gpurun_out/r02t_bd_mulv24.txt gpurun_out/r02t_mem_lenet.txt
