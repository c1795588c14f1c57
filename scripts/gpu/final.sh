# round-end verification: tests, smoke, both bench arms, launch list, ncu of the top kernel
mkdir -p gpurun_out
TAG=${1:-final}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --impl reference > gpurun_out/ref_$TAG.log 2>&1; echo "ref exit $?" >> gpurun_out/ref_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-steps 1 > gpurun_out/ncu_l_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_conv_sqsum --launch-skip 4 -c 1 \
    -o gpurun_out/prof_conv2_$TAG -f python bench.py --profile-steps 1 > gpurun_out/ncu_f_$TAG.log 2>&1
tail -2 gpurun_out/gpu_tests_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log; tail -1 gpurun_out/bench_$TAG.log; tail -1 gpurun_out/ref_$TAG.log
