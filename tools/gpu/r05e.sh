mkdir -p gpurun_out; set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gr_matmul_q_kernel<4>" --launch-skip 1 -c 1 -o gpurun_out/r05e_q python tools/host_gpu_lag.py 25 mulv > gpurun_out/r05e_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gr_matmul2_db_kernel" -c 3 -o gpurun_out/r05e_db python tools/host_gpu_lag.py 25 mulv > gpurun_out/r05e_ncu2.log 2>&1
