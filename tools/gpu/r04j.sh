timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lane16_fold" --launch-skip 3 -c 1 -o gpurun_out/r04j_fold python tools/vfy_split.py 20 > gpurun_out/r04j_ncu.log 2>&1
tail -1 gpurun_out/r04j_ncu.log
