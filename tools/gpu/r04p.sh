timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py tests/test_gpu_sessions.py -x -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 900 python bench.py --relu-sweep-log2n 0 --matmul-n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep 20 --mulv-variants "" --no-cpu-baseline --no-step-profile 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['relu']
print(d['value'], r['exec_ms'], r['verified_ms'], [(p['log2n'], p['ms']) for p in d['mulv_sweep']['points']])"; done
