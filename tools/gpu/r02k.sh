mkdir -p gpurun_out
for a in "20 mulv" "22 mulv" "16 relu" "14 relu"; do timeout 300 python tools/host_split.py $a; done > gpurun_out/r02k_split.txt 2>&1
