mkdir -p gpurun_out
timeout 300 python tools/breakdown.py --prog mulv --log2n 25 --d 64 > gpurun_out/r03e_bd_mulv25.txt 2>&1
timeout 300 python tools/host_gpu_lag.py 25 mulv > gpurun_out/r03e_lag25.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"base_fold_tc_kernel" --launch-skip 3 -c 1 -o gpurun_out/r03e_base_fold_q8 python tools/host_gpu_lag.py 25 mulv > gpurun_out/r03e_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gfv_line_kernel|gfv_base_kernel" --launch-skip 30 -c 3 -o gpurun_out/r03e_gfv python tools/vfy_split.py 20 > gpurun_out/r03e_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"line_b_kernel" --launch-skip 6 -c 2 -o gpurun_out/r03e_line_b8 python tools/host_gpu_lag.py 25 mulv > gpurun_out/r03e_ncu3.log 2>&1
head -24 gpurun_out/r03e_bd_mulv25.txt; head -3 gpurun_out/r03e_lag25.txt; tail -3 gpurun_out/r03e_ncu*.log; ls -la gpurun_out/*.ncu-rep
