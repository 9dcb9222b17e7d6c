timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "matmul_q or k16" > gpurun_out/v.log 2>&1; tail -1 gpurun_out/v.log
for q in 4 2; do R3_TABLE_Q=$q timeout 600 python tools/breakdown.py --log2n 25 2>&1 | grep -E "step|matmul_q|k16|line_b "; done
