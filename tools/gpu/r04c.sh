mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gr_matmul_q_kernel|line_b_kernel" --launch-skip 6 -c 3 -o gpurun_out/r04c_tables python tools/host_gpu_lag.py 25 mulv > gpurun_out/r04c_ncu.log 2>&1
tail -3 gpurun_out/r04c_ncu.log
