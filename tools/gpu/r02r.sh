mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k gfv -x -q -p no:cacheprovider > gpurun_out/r02r_k.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_k.log
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py -x -q -p no:cacheprovider > gpurun_out/r02r_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_golden.log
for n in 16 20; do timeout 300 python tools/vfy_split.py $n; done > gpurun_out/r02r_vsplit.txt 2>&1
tail -30 gpurun_out/r02r_k.log; tail -5 gpurun_out/r02r_golden.log; cat gpurun_out/r02r_vsplit.txt
