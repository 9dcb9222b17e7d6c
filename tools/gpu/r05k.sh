mkdir -p gpurun_out; set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r05k_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r05k_pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r05k_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r05k_smoke.log
timeout 1800 python bench.py > gpurun_out/r05k_bench.json 2> gpurun_out/r05k_bench.err; echo "bench rc=$?" >> gpurun_out/r05k_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r05k_launches.csv python bench.py --steps 2 --warmup 1 --relu-log2n 0 --relu-sweep-log2n 0 --matmul-n 0 --mlp-batch 0 --lenet-batch 0 --mulv-sweep "" --no-cpu-baseline --no-step-profile > /dev/null 2>&1
gzip -f gpurun_out/r05k_launches.csv
timeout 1800 python bench.py --impl reference > gpurun_out/r05k_ref.json 2> gpurun_out/r05k_ref.err
tail -3 gpurun_out/r05k_pytest.log; tail -2 gpurun_out/r05k_smoke.log; tail -c 300 gpurun_out/r05k_bench.err
