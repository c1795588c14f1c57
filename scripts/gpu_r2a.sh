mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc5.py -x -q -s > gpurun_out/tc5.log 2>&1; echo "exit $?" >> gpurun_out/tc5.log
tail -15 gpurun_out/tc5.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "exit $?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
