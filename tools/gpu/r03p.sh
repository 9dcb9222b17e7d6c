mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py tests/test_gpu_golden_scale.py tests/test_gpu_sessions.py -x -q -p no:cacheprovider > gpurun_out/r03p_t.log 2>&1; echo "rc=$?" >> gpurun_out/r03p_t.log
tail -2 gpurun_out/r03p_t.log; grep -E "^E |FAILED" gpurun_out/r03p_t.log | head -5
timeout 300 python tools/breakdown.py --prog mulv --log2n 25 --d 64 2>&1 | head -12
timeout 300 python tools/vfy_split.py 20 2>&1 | head -20
