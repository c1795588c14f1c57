# bootstrapping GPU tests (+ the lincomb_plain / CBC tests it touches), per-op timing, bench line
mkdir -p gpurun_out
TAG=${1:-b1}
timeout 1500 python -m pytest tests/test_gpu_bootstrap.py tests/test_gpu_pipeline.py -m gpu -x -q -s > gpurun_out/boot_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/boot_$TAG.log
for r in boot12 boot16s; do timeout 600 python scripts/time_bootstrap.py $r; done >> gpurun_out/boot_$TAG.log 2>&1
timeout 600 python bench.py --workload boot >> gpurun_out/boot_$TAG.log 2>&1
tail -45 gpurun_out/boot_$TAG.log
