mkdir -p gpurun_out; set -x
timeout 1500 python bench.py > gpurun_out/r03c_bench.json 2> gpurun_out/r03c_bench.err; echo "bench rc=$?" >> gpurun_out/r03c_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03c_launches.csv python bench.py --steps 2 --warmup 1 --relu-log2n 0 --relu-sweep-log2n 0 --matmul-n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep "" --no-cpu-baseline --no-step-profile > /dev/null 2>&1
gzip -f gpurun_out/r03c_launches.csv
tail -c 400 gpurun_out/r03c_bench.err
