mkdir -p gpurun_out; set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02p_pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r02p_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02p_smoke.log
timeout 1500 python bench.py > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err; echo "bench rc=$?" >> gpurun_out/r02p_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02p_ref.json 2> gpurun_out/r02p_ref.err; echo "ref rc=$?" >> gpurun_out/r02p_ref.err
tail -3 gpurun_out/r02p_pytest.log; tail -2 gpurun_out/r02p_smoke.log; tail -c 1500 gpurun_out/r02p_bench.json; cat gpurun_out/r02p_ref.json
