mkdir -p gpurun_out
for b in 128 256 384; do timeout 600 python tools/mem_probe.py lenet $b 2>&1 | tail -1; done > gpurun_out/r03a_mem_lenet.txt 2>&1
cat gpurun_out/r03a_mem_lenet.txt | cut -c1-400
