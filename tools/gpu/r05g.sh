mkdir -p gpurun_out; set -x
L=paper_2411_09287_b200
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider -k "matmul" > gpurun_out/r05g_ktests.log 2>&1; echo "rc=$?" >> gpurun_out/r05g_ktests.log
B="--relu-log2n 0 --relu-sweep-log2n 0 --matmul-n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep '' --mulv-variants '' --no-cpu-baseline"
cp $L/libr3b200.so /tmp/new.so
for v in new old new old; do
  cp $L/libr3b200_$v.so $L/libr3b200.so 2>/dev/null || cp /tmp/new.so $L/libr3b200.so
  eval timeout 600 python bench.py $B > gpurun_out/r05g_bench_$v.json 2> gpurun_out/r05g_bench_$v.err
  python -c "import json;d=json.load(open('gpurun_out/r05g_bench_$v.json'));print('$v',d['value'],d['ms_per_step'],d['roofline']['frac'],[(t['entry_point'],round(t['ms'],3)) for t in d['step_kernels']['top']])" >> gpurun_out/r05g_summary.txt 2>&1
done
cat gpurun_out/r05g_summary.txt
