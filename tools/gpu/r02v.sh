mkdir -p gpurun_out
(timeout 300 python tools/host_gpu_lag.py 24 mulv; timeout 300 python tools/host_gpu_lag.py 20 mulv; timeout 300 python tools/host_gpu_lag.py 16 relu) > gpurun_out/r02v_lag.txt 2>&1
cat gpurun_out/r02v_lag.txt
