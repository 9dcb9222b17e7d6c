mkdir -p gpurun_out
timeout 300 python tools/host_cprofile.py mulv 20 tottime > gpurun_out/r02g_mulv_tottime.txt 2>&1
timeout 300 python tools/host_cprofile.py mulv 20 cumulative > gpurun_out/r02g_mulv_cum.txt 2>&1
timeout 300 python tools/host_cprofile.py relu_v 16 tottime > gpurun_out/r02g_reluv_tottime.txt 2>&1
timeout 300 python tools/host_cprofile.py relu_v 16 cumulative > gpurun_out/r02g_reluv_cum.txt 2>&1
timeout 300 python tools/host_cprofile.py relu 16 tottime > gpurun_out/r02g_relu_tottime.txt 2>&1
