mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rotate" > gpurun_out/t_rot.log 2>&1; echo "exit $?" >> gpurun_out/t_rot.log
tail -3 gpurun_out/t_rot.log
