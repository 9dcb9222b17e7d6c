mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_sessions.py tests/test_gpu_circuit.py -x -q -p no:cacheprovider > gpurun_out/r03d_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r03d_golden.log
timeout 300 python tools/party_cprofile.py mulv 20 tottime 1 > gpurun_out/r03d_pcp_mulv.txt 2>&1
timeout 300 python tools/party_cprofile.py relu_v 16 tottime 1 > gpurun_out/r03d_pcp_relu.txt 2>&1
for L in 24 25; do timeout 600 python bench.py --log2n $L --no-cpu-baseline --relu-sweep-log2n 0 --mlp-batch 0 --lenet-batch 0 --matmul-n 0 --mulv-sweep "" > gpurun_out/r03d_bench$L.json 2> gpurun_out/r03d_bench$L.err; done
tail -3 gpurun_out/r03d_golden.log
for L in 24 25; do python - $L <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/r03d_bench{sys.argv[1]}.json').read().strip().splitlines()[-1])
print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['per_party_rate']['value'], d['relu']['exec_ms'], d['relu']['verified_ms'])
PY
done
head -50 gpurun_out/r03d_pcp_mulv.txt
