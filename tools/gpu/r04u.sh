timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gr_matmul_q_kernel" --launch-skip 8 -c 1 -o gpurun_out/r04u_q python tools/host_gpu_lag.py 25 mulv > gpurun_out/r04u_ncu.log 2>&1
tail -1 gpurun_out/r04u_ncu.log
