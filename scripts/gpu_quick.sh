mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 900 python scripts/bench_primitives.py > gpurun_out/prims.log 2>&1
tail -1 gpurun_out/prims.log
