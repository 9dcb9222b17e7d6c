mkdir -p gpurun_out; set -x
timeout 300 python tools/host_cprofile.py relu 16 tottime > gpurun_out/r05b_cprof_relu.txt 2>&1
timeout 300 python tools/host_cprofile.py relu 16 cumtime > gpurun_out/r05b_cprof_relu_cum.txt 2>&1
timeout 300 python tools/call_sites.py relu 16 > gpurun_out/r05b_sites_relu.txt 2>&1
timeout 300 python tools/host_cprofile.py relu_v 16 tottime > gpurun_out/r05b_cprof_reluv.txt 2>&1
timeout 300 python tools/call_sites.py relu_check 16 > gpurun_out/r05b_sites_reluv.txt 2>&1
