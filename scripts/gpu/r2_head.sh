# state of HEAD: gpu tests, tcgen05 conv timings, bench (short)
mkdir -p gpurun_out
TAG=${1:-head}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
timeout 600 python scripts/time_convtc.py 3 > gpurun_out/time_convtc_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/time_convtc_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-steps 1 > gpurun_out/ncu_l_$TAG.log 2>&1
tail -3 gpurun_out/gpu_tests_$TAG.log; cat gpurun_out/time_convtc_$TAG.log | tail -20; tail -c 1500 gpurun_out/bench_$TAG.log
