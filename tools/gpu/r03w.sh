mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "base_fold_q4" -x -q -p no:cacheprovider > gpurun_out/r03w_k.log 2>&1; echo "rc=$?" >> gpurun_out/r03w_k.log
tail -3 gpurun_out/r03w_k.log; grep -E "^E |FAILED|Timeout" gpurun_out/r03w_k.log | head -8
