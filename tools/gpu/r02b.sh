mkdir -p gpurun_out
timeout 300 python tools/lf_bench.py > gpurun_out/r02b_lf.txt 2>&1; echo "rc=$?" >> gpurun_out/r02b_lf.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_golden_scale.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r02b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_pytest.log
timeout 600 python bench.py --no-cpu-baseline --relu-log2n 0 --relu-sweep-log2n 0 --matmul-n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep "" > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
cat gpurun_out/r02b_lf.txt; tail -3 gpurun_out/r02b_pytest.log
