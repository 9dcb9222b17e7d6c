mkdir -p gpurun_out; set -x
timeout 600 python bench.py --relu-log2n 0 --relu-sweep-log2n 0 --matmul-n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep '' --mulv-variants '' --no-cpu-baseline > gpurun_out/r05h_bench.json 2> gpurun_out/r05h_bench.err; echo "rc=$?" >> gpurun_out/r05h_bench.err
python -c "import json;d=json.load(open('gpurun_out/r05h_bench.json'));print(json.dumps(d['roofline_step_top']));print(json.dumps(d['step_kernels']['top'][:2]))"
