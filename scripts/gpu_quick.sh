mkdir -p gpurun_out
for args in "3 4 0 14" "3 8 0 14"; do
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/probe_conv.py $args 2>&1 | grep -E "cfg|rror" | head -2
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv_square_sum" 2>&1 | tail -2
timeout 300 python scripts/time_convsq.py 3 2>&1 | tail -3
