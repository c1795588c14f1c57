# round-2 verification: every GPU test, smoke, both bench arms (driver defaults), launch list,
# one ncu --set full capture of the top kernel inside bench.py
mkdir -p gpurun_out
TAG=${1:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_$TAG.log 2>&1; echo "ref exit $?" >> gpurun_out/ref_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-steps 1 > gpurun_out/ncu_l_$TAG.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_convtc_p16 -c 1 \
    -o gpurun_out/prof_conv2_$TAG -f python bench.py --profile-steps 1 > gpurun_out/ncu_f_$TAG.log 2>&1
tail -2 gpurun_out/gpu_tests_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log; tail -c 400 gpurun_out/bench_$TAG.log; tail -c 300 gpurun_out/ref_$TAG.log
