mkdir -p gpurun_out
for b in 128 256 512; do timeout 600 python tools/mem_probe.py lenet $b 2>&1 | tail -4; done
