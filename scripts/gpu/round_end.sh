#!/bin/bash
# One GPU session: gpu tests, bench, then the ncu recipe (scripts/prof_bench.sh).
TAG=${1:-cur}
KREGEX=${2:-k_conv_sqsum}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 1200 bash scripts/prof_bench.sh $TAG "$KREGEX" 2; echo "prof exit $?" >> gpurun_out/bench_$TAG.log
tail -3 gpurun_out/gpu_tests_$TAG.log; tail -2 gpurun_out/bench_$TAG.log
