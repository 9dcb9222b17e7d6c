mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_golden.py tests/test_gpu_golden_scale.py tests/test_gpu_sessions.py tests/test_gpu_circuit.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/r03r_t.log 2>&1; echo "rc=$?" >> gpurun_out/r03r_t.log
tail -2 gpurun_out/r03r_t.log; grep -E "^E |FAILED|Error" gpurun_out/r03r_t.log | head -12
timeout 300 python tools/level_cost.py mulv 20 2>&1 | head -8
timeout 300 python tools/level_cost.py relu 16 2>&1 | head -8
timeout 600 python bench.py --no-cpu-baseline --relu-sweep-log2n 0 --mlp-batch 0 --lenet-batch 0 --matmul-n 0 --mulv-sweep "20" --mulv-variants "" > gpurun_out/r03r_bench.json 2> gpurun_out/r03r_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r03r_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'], d['relu']['exec_ms'], d['relu']['verified_ms'], d['mulv_sweep']['points'])
PY
