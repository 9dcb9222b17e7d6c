timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "lane16" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lane16" --launch-skip 6 -c 2 -o gpurun_out/r04i_lane16 python tools/vfy_split.py 20 > gpurun_out/r04i_ncu.log 2>&1
tail -2 gpurun_out/r04i_ncu.log
