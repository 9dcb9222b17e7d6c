mkdir -p gpurun_out
timeout 300 python tools/call_sites.py relu_check 16 > gpurun_out/r02i_sites_relu.txt 2>&1
timeout 300 python tools/call_sites.py mulv 20 > gpurun_out/r02i_sites_mulv.txt 2>&1
