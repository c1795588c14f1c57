mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv_square_sum" > gpurun_out/t_conv.log 2>&1; echo "exit $?" >> gpurun_out/t_conv.log
timeout 300 python scripts/time_convsq.py 3 > gpurun_out/tconv.log 2>&1
tail -2 gpurun_out/t_conv.log; cat gpurun_out/tconv.log | tail -4
