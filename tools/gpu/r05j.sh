mkdir -p gpurun_out; set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 1800 python bench.py > gpurun_out/r05j_bench.json 2> gpurun_out/r05j_bench.err; echo "bench rc=$?" >> gpurun_out/r05j_bench.err
tail -c 400 gpurun_out/r05j_bench.err
