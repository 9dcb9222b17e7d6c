mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02j_pytest.log
timeout 600 python bench.py --no-cpu-baseline --relu-sweep-log2n 20 --mlp-batch 0 --lenet-batch 0 --matmul-n 0 --no-step-profile > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err
timeout 300 python tools/call_sites.py relu_check 16 > gpurun_out/r02j_sites_relu.txt 2>&1
tail -3 gpurun_out/r02j_pytest.log
