mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plainops.py -x -q -k p15 > gpurun_out/p15.log 2>&1; echo "exit $?" >> gpurun_out/p15.log
tail -30 gpurun_out/p15.log
