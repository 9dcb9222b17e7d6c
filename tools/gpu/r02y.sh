mkdir -p gpurun_out
timeout 300 python tools/host_cprofile.py mulv 20 tottime > gpurun_out/r02y_cp_tot.txt 2>&1
timeout 300 python tools/host_cprofile.py mulv 20 cumtime > gpurun_out/r02y_cp_cum.txt 2>&1
timeout 300 python tools/host_cprofile.py relu_v 16 tottime > gpurun_out/r02y_cp_relu_tot.txt 2>&1
head -80 gpurun_out/r02y_cp_tot.txt
