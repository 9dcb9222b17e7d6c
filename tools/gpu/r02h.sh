mkdir -p gpurun_out
timeout 300 python tools/party_cprofile.py mulv 20 tottime 50 > gpurun_out/r02h_mulv_party.txt 2>&1
timeout 300 python tools/party_cprofile.py relu_v 16 tottime 60 > gpurun_out/r02h_reluv_party.txt 2>&1
timeout 300 python tools/party_cprofile.py relu_v 16 cumulative 80 > gpurun_out/r02h_reluv_party_cum.txt 2>&1
