mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "base_fold" -x -q -p no:cacheprovider > gpurun_out/r03j_k.log 2>&1; echo "rc=$?" >> gpurun_out/r03j_k.log
timeout 900 python -m pytest tests/test_gpu_sessions.py tests/test_gpu_golden_scale.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/r03j_s.log 2>&1; echo "rc=$?" >> gpurun_out/r03j_s.log
timeout 300 python tools/breakdown.py --prog mulv --log2n 25 --d 64 > gpurun_out/r03j_bd_mulv25.txt 2>&1
tail -3 gpurun_out/r03j_k.log; grep -E "^E |FAILED" gpurun_out/r03j_k.log | head; tail -3 gpurun_out/r03j_s.log; grep -E "^E |FAILED" gpurun_out/r03j_s.log | head; head -14 gpurun_out/r03j_bd_mulv25.txt
