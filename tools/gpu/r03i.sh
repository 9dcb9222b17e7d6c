mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_golden_scale.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/r03i_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r03i_golden.log
timeout 300 python tools/breakdown.py --prog mulv --log2n 25 --d 64 > gpurun_out/r03i_bd_mulv25.txt 2>&1
tail -3 gpurun_out/r03i_golden.log; head -10 gpurun_out/r03i_bd_mulv25.txt
