mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/r03h_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r03h_golden.log
timeout 300 python tools/vfy_split.py 20 > gpurun_out/r03h_vsplit.txt 2>&1
tail -3 gpurun_out/r03h_golden.log; head -12 gpurun_out/r03h_vsplit.txt
