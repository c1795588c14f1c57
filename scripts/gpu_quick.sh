mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_networks.py -m gpu -x -q -k "cbc" > gpurun_out/t_cbc.log 2>&1; echo "exit $?" >> gpurun_out/t_cbc.log
tail -25 gpurun_out/t_cbc.log
