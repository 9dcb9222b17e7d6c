mkdir -p gpurun_out; set -x
timeout 900 python bench.py --log2n 20 --steps 3 --warmup 3 --e2e-steps 2 --relu-log2n 0 --relu-sweep-log2n 0 --matmul-n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep 27 --mulv-variants '' --no-cpu-baseline --no-step-profile > gpurun_out/r05i_bench27.json 2> gpurun_out/r05i_bench27.err; echo "rc=$?" >> gpurun_out/r05i_bench27.err
tail -c 600 gpurun_out/r05i_bench27.err
python -c "import json;d=json.load(open('gpurun_out/r05i_bench27.json'));print(json.dumps(d['mulv_sweep']))"
nvidia-smi --query-gpu=memory.total --format=csv
