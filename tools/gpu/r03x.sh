mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sessions.py tests/test_gpu_golden.py tests/test_gpu_golden_scale.py tests/test_gpu_scale.py tests/test_gpu_circuit.py -x -q -p no:cacheprovider > gpurun_out/r03x_t.log 2>&1; echo "rc=$?" >> gpurun_out/r03x_t.log
tail -2 gpurun_out/r03x_t.log; grep -E "^E |FAILED|Error" gpurun_out/r03x_t.log | head -8
timeout 300 python tools/vfy_split.py 20 2>&1 | head -8
timeout 600 python tools/ppml_breakdown.py mlp 4096 check 2>&1 | head -6
