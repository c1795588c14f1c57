mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_convtc.py tests/test_gpu_tc5.py -x -q > gpurun_out/convtc.log 2>&1; echo "exit $?" >> gpurun_out/convtc.log
timeout 600 python scripts/time_convtc.py 3 > gpurun_out/time_convtc.log 2>&1; echo "exit $?" >> gpurun_out/time_convtc.log
timeout 600 python scripts/role_convtc.py > gpurun_out/role_convtc.log 2>&1; echo "exit $?" >> gpurun_out/role_convtc.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "exit $?" >> gpurun_out/bench.log
tail -3 gpurun_out/convtc.log; cat gpurun_out/time_convtc.log gpurun_out/role_convtc.log; tail -c 3000 gpurun_out/bench.log
