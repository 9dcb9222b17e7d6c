mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --relu-log2n 0 --relu-sweep-log2n 0 --mlp-batch 0 --lenet-batch 0 --matmul-n 0 --mulv-sweep "" > gpurun_out/r03s_bench.json 2> gpurun_out/r03s_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r03s_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])
PY
for r in 512 1024; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-step-profile --relu-log2n 0 --relu-sweep-log2n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep "" --matmul-verified-rows $r > gpurun_out/r03s_mm$r.json 2> gpurun_out/r03s_mm$r.err; python - $r <<'PY'
import json,sys
try:
    d=json.loads(open(f'gpurun_out/r03s_mm{sys.argv[1]}.json').read().strip().splitlines()[-1])
    print(sys.argv[1], d['matmul']['verified'])
except Exception as e:
    print(sys.argv[1], 'fail', e)
PY
tail -2 gpurun_out/r03s_mm$r.err; done
