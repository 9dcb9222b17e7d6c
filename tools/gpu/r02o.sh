mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02o_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02o_pytest.log
for a in "20 mulv" "16 relu"; do timeout 300 python tools/host_split.py $a; done > gpurun_out/r02o_split.txt 2>&1
tail -3 gpurun_out/r02o_pytest.log
