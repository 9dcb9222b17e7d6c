timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py tests/test_gpu_sessions.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/w.log 2>&1; tail -1 gpurun_out/w.log
timeout 900 python bench.py --log2n 20 --matmul-n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep "" --mulv-variants "" --no-cpu-baseline --no-step-profile 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['relu']; s=d['relu_sweep']
print(r['exec_ms'], r['verified_ms'], s['exec_ms'], s['verified_ms'], s['exec_kernels']['device_busy_ms'])"
