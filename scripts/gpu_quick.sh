mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv_square_sum" > gpurun_out/t.log 2>&1; echo "exit $?" >> gpurun_out/t.log
grep -E "passed|failed|exit|Error" gpurun_out/t.log | tail -4
timeout 300 python scripts/time_convsq.py 3 2>&1 | tail -3
