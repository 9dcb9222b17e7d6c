mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "base_fold" -x -q -p no:cacheprovider > gpurun_out/r03f_k.log 2>&1; echo "rc=$?" >> gpurun_out/r03f_k.log
timeout 1200 python -m pytest tests/test_gpu_golden_scale.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/r03f_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r03f_golden.log
timeout 300 python tools/breakdown.py --prog mulv --log2n 25 --d 64 > gpurun_out/r03f_bd_mulv25.txt 2>&1
tail -3 gpurun_out/r03f_k.log; tail -3 gpurun_out/r03f_golden.log; head -8 gpurun_out/r03f_bd_mulv25.txt
