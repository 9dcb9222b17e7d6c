mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "base_fold" -x -q -p no:cacheprovider > gpurun_out/r02u_k.log 2>&1; echo "rc=$?" >> gpurun_out/r02u_k.log
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/r02u_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r02u_golden.log
timeout 300 python tools/breakdown.py --prog mulv --log2n 24 --d 64 > gpurun_out/r02u_bd_mulv24.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --relu-log2n 0 --relu-sweep-log2n 0 --mlp-batch 0 --lenet-batch 0 --matmul-n 0 --mulv-sweep "" > gpurun_out/r02u_bench.json 2> gpurun_out/r02u_bench.err
tail -30 gpurun_out/r02u_k.log; tail -30 gpurun_out/r02u_golden.log; head -30 gpurun_out/r02u_bd_mulv24.txt; tail -c 600 gpurun_out/r02u_bench.json; tail -5 gpurun_out/r02u_bench.err
