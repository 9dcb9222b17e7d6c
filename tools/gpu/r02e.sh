mkdir -p gpurun_out
timeout 300 python tools/lf_bench.py > gpurun_out/r02e_lf.txt 2>&1; echo "rc=$?" >> gpurun_out/r02e_lf.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02e_pytest.log
timeout 600 python bench.py --no-cpu-baseline --relu-sweep-log2n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep "" > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
cat gpurun_out/r02e_lf.txt; tail -3 gpurun_out/r02e_pytest.log
