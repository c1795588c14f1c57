# quick verification of the tree: every GPU test, smoke, default bench line
mkdir -p gpurun_out
TAG=${1:-verify}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
tail -3 gpurun_out/gpu_tests_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log; tail -c 1500 gpurun_out/bench_$TAG.log
