mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_fold_tc -s 11 -c 1 -o gpurun_out/r02c_lf python tools/lf_bench.py 4194304 > gpurun_out/r02c_ncu.txt 2>&1
echo rc=$? >> gpurun_out/r02c_ncu.txt
tail -5 gpurun_out/r02c_ncu.txt
