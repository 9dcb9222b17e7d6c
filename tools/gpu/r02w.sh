mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py tests/test_gpu_sessions.py -x -q -p no:cacheprovider > gpurun_out/r02w_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r02w_golden.log
(timeout 300 python tools/host_gpu_lag.py 24 mulv; timeout 300 python tools/host_gpu_lag.py 20 relu) > gpurun_out/r02w_lag.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --relu-sweep-log2n 0 --mlp-batch 0 --lenet-batch 0 --matmul-n 0 --mulv-sweep "" > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err
tail -3 gpurun_out/r02w_golden.log; head -12 gpurun_out/r02w_lag.txt; grep -A3 "relu 2" gpurun_out/r02w_lag.txt; tail -c 300 gpurun_out/r02w_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02w_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])
r=d['relu']; print('relu', r['exec_ms'], r['verified_ms'])
PY
