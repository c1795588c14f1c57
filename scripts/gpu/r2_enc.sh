mkdir -p gpurun_out
timeout 600 python scripts/time_encrypt.py > gpurun_out/time_enc.log 2>&1; tail -5 gpurun_out/time_enc.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plainops.py -x -q -k "encrypt or encode or plain" > gpurun_out/enc_par.log 2>&1; tail -1 gpurun_out/enc_par.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_enc.csv python scripts/time_encrypt.py 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_enc.csv 2>/dev/null | head -12
