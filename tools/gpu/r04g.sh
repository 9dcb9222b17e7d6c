mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r04g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r04g_pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r04g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r04g_smoke.log
tail -3 gpurun_out/r04g_pytest.log; tail -2 gpurun_out/r04g_smoke.log
