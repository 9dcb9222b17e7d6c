mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline --relu-sweep-log2n 0 --mlp-batch 0 --lenet-batch 0 --matmul-n 0 --mulv-sweep "" > gpurun_out/r03n_bench.json 2> gpurun_out/r03n_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r03n_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['e2e']['value'], d['per_party_rate']['value'], d['relu']['exec_ms'], d['relu']['verified_ms'])
print(json.dumps(d['step_kernels']['top'])[:1500])
PY
