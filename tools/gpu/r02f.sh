mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_pytest.log
timeout 600 python bench.py --no-cpu-baseline --relu-sweep-log2n 0 --mlp-batch 0 --lenet-batch 0 --matmul-n 0 > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
tail -3 gpurun_out/r02f_pytest.log
