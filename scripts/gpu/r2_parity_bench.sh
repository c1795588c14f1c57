mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/mb_fp64_occ.cu -o /tmp/mb_fp64_occ && /tmp/mb_fp64_occ > gpurun_out/mb_fp64_occ.log 2>&1
timeout 900 python -m pytest tests/test_gpu_convtc.py -x -q > gpurun_out/convtc.log 2>&1; echo "exit $?" >> gpurun_out/convtc.log
timeout 1500 python -m pytest tests/test_gpu_networks.py -x -q -k carry_plan > gpurun_out/carry.log 2>&1; echo "exit $?" >> gpurun_out/carry.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "exit $?" >> gpurun_out/bench.log
tail -3 gpurun_out/convtc.log; tail -30 gpurun_out/carry.log; cat gpurun_out/mb_fp64_occ.log; head -c 700 gpurun_out/bench.log; grep -o '"breakdown.*' gpurun_out/bench.log | head -c 1500
