mkdir -p gpurun_out
timeout 300 python tools/lf_bench.py > gpurun_out/r02d_lf.txt 2>&1; echo "rc=$?" >> gpurun_out/r02d_lf.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -k level_fold -m gpu -x -q -p no:cacheprovider > gpurun_out/r02d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_pytest.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_fold_tc -s 11 -c 1 -o gpurun_out/r02d_lf python tools/lf_bench.py 4194304 > gpurun_out/r02d_ncu.txt 2>&1
cat gpurun_out/r02d_lf.txt; tail -3 gpurun_out/r02d_pytest.log
