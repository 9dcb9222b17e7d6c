mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py -x -q -p no:cacheprovider > gpurun_out/r03b_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r03b_golden.log
for b in 128 192 256; do timeout 600 python tools/mem_probe.py lenet $b 2>&1 | tail -1 | grep -o "lenet [0-9]*\|'peak_gib': [0-9.]*\|OutOfMemory"; done > gpurun_out/r03b_mem_lenet.txt 2>&1
tail -3 gpurun_out/r03b_golden.log; cat gpurun_out/r03b_mem_lenet.txt
