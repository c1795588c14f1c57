mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_convtc.py -x -q > gpurun_out/convtc.log 2>&1; echo "exit $?" >> gpurun_out/convtc.log
tail -25 gpurun_out/convtc.log
