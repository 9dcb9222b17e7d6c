mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "level_fold" -x -q -p no:cacheprovider > gpurun_out/r03v_k.log 2>&1; echo "rc=$?" >> gpurun_out/r03v_k.log
timeout 900 python -m pytest tests/test_gpu_golden_scale.py tests/test_gpu_sessions.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/r03v_s.log 2>&1; echo "rc=$?" >> gpurun_out/r03v_s.log
tail -2 gpurun_out/r03v_k.log; grep -E "^E |FAILED" gpurun_out/r03v_k.log | head -5; tail -2 gpurun_out/r03v_s.log; grep -E "^E |FAILED" gpurun_out/r03v_s.log | head
timeout 300 python tools/breakdown.py --prog mulv --log2n 25 --d 64 2>&1 | head -8
