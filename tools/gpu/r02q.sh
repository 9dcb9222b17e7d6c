mkdir -p gpurun_out
for n in 16 20; do timeout 300 python tools/vfy_split.py $n; done > gpurun_out/r02q_vsplit.txt 2>&1
for a in "20 mulv" "16 relu"; do timeout 300 python tools/host_split.py $a; done > gpurun_out/r02q_split.txt 2>&1
timeout 300 python tools/breakdown.py --prog relu --log2n 16 > gpurun_out/r02q_bd_relu16.txt 2>&1
timeout 300 python tools/breakdown.py --prog mulv --log2n 20 > gpurun_out/r02q_bd_mulv20.txt 2>&1
cat gpurun_out/r02q_vsplit.txt gpurun_out/r02q_split.txt | head -150
