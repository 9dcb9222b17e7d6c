timeout 900 ncu --set full --clock-control none --import-source on -k regex:"level_fold_tc_kernel|gr_matmul2_db_kernel|gr_matmul_q_kernel" --launch-skip 40 -c 6 -o gpurun_out/r04r_tail python tools/host_gpu_lag.py 25 mulv > gpurun_out/r04r_ncu.log 2>&1
tail -1 gpurun_out/r04r_ncu.log
