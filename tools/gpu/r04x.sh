mkdir -p gpurun_out; set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r04x_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r04x_pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r04x_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r04x_smoke.log
timeout 1800 python bench.py > gpurun_out/r04x_bench.json 2> gpurun_out/r04x_bench.err; echo "bench rc=$?" >> gpurun_out/r04x_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r04x_launches.csv python bench.py --steps 2 --warmup 1 --relu-log2n 0 --relu-sweep-log2n 0 --matmul-n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep "" --no-cpu-baseline --no-step-profile > /dev/null 2>&1
gzip -f gpurun_out/r04x_launches.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"base_fold_tc_kernel" --launch-skip 3 -c 1 -o gpurun_out/r04x_base_fold_q16 python tools/host_gpu_lag.py 25 mulv > gpurun_out/r04x_ncu1.log 2>&1
tail -3 gpurun_out/r04x_pytest.log; tail -2 gpurun_out/r04x_smoke.log; tail -c 300 gpurun_out/r04x_bench.err
