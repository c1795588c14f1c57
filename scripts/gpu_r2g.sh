mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_convtc.py -x -q > gpurun_out/convtc.log 2>&1; echo "exit $?" >> gpurun_out/convtc.log
tail -15 gpurun_out/convtc.log
timeout 600 python scripts/time_convtc.py 3 > gpurun_out/time_convtc5.log 2>&1; echo "exit $?" >> gpurun_out/time_convtc5.log
cat gpurun_out/time_convtc5.log
