mkdir -p gpurun_out
timeout 300 python scripts/time_encrypt.py 1 > gpurun_out/time_enc.log 2>&1; tail -3 gpurun_out/time_enc.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_enc16 -s 2 -c 2 -f -o gpurun_out/ncu_enc16_s6 python scripts/time_encrypt.py 1 > gpurun_out/ncu_enc.log 2>&1
tail -2 gpurun_out/ncu_enc.log
