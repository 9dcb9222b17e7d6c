mkdir -p gpurun_out
timeout 600 python tools/mem_probe.py lenet 64 > gpurun_out/r02m_mem_lenet64.txt 2>&1
timeout 600 python tools/mem_probe.py relu 262144 > gpurun_out/r02m_mem_relu18.txt 2>&1
