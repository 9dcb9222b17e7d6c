mkdir -p gpurun_out
timeout 300 python tools/host_sampler.py mulv 20 20 > gpurun_out/r02z_samp_mulv.txt 2>&1
timeout 300 python tools/host_sampler.py relu_v 16 10 > gpurun_out/r02z_samp_relu.txt 2>&1
cat gpurun_out/r02z_samp_mulv.txt
