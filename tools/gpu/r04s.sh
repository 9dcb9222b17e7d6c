timeout 900 ncu --set full --clock-control none --import-source on -k regex:"level_fold_tc_kernel|gr_matmul2_db_kernel" --launch-skip 25 -c 2 -o gpurun_out/r04s_big python tools/host_gpu_lag.py 25 mulv > gpurun_out/r04s_ncu.log 2>&1
tail -1 gpurun_out/r04s_ncu.log
