mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "dot_log_folds" -x -q -p no:cacheprovider > gpurun_out/r03g_k.log 2>&1; echo "rc=$?" >> gpurun_out/r03g_k.log
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py -x -q -p no:cacheprovider > gpurun_out/r03g_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r03g_golden.log
timeout 300 python tools/vfy_split.py 20 > gpurun_out/r03g_vsplit.txt 2>&1
tail -3 gpurun_out/r03g_k.log; grep -E "Error|assert" gpurun_out/r03g_k.log | head -5; tail -3 gpurun_out/r03g_golden.log; cat gpurun_out/r03g_vsplit.txt
