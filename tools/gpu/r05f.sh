mkdir -p gpurun_out; set -x
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gr_matmul_q_kernel<.int.4>" --launch-skip 1 -c 1 -o gpurun_out/r05f_q python tools/host_gpu_lag.py 25 mulv > gpurun_out/r05f_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gr_matmul2_db_kernel" -s 2 -c 1 -o gpurun_out/r05f_db python tools/prof_targets2.py line > gpurun_out/r05f_ncu2.log 2>&1
