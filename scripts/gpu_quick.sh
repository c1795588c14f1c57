mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_networks.py -m gpu -x -q > gpurun_out/t.log 2>&1; echo "exit $?" >> gpurun_out/t.log
grep -E "passed|failed|exit" gpurun_out/t.log | tail -3
