mkdir -p gpurun_out; set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gr_matmul_q_kernel" --launch-skip 4 -c 1 -o gpurun_out/r05d_q python tools/host_gpu_lag.py 25 mulv > gpurun_out/r05d_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gr_matmul2_db_kernel" --launch-skip 40 -c 1 -o gpurun_out/r05d_db python tools/host_gpu_lag.py 25 mulv > gpurun_out/r05d_ncu2.log 2>&1
ls -la gpurun_out
