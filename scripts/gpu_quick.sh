mkdir -p gpurun_out
timeout 900 python scripts/bench_primitives.py > gpurun_out/prims.log 2>&1
tail -1 gpurun_out/prims.log
