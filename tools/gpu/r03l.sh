mkdir -p gpurun_out
for b in 8 16; do R3_BASE_BLOCK=$b timeout 300 python tools/breakdown.py --prog mulv --log2n 25 --d 64 2>&1 | head -6; done
