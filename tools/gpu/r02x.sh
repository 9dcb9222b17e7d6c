mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "base_fold" -x -q -p no:cacheprovider > gpurun_out/r02x_k.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_k.log
timeout 300 python tools/breakdown.py --prog mulv --log2n 24 --d 64 > gpurun_out/r02x_bd_mulv24.txt 2>&1
tail -3 gpurun_out/r02x_k.log; head -12 gpurun_out/r02x_bd_mulv24.txt
