# bootstrapping GPU tests (+ the lincomb_plain / CBC tests it touches)
mkdir -p gpurun_out
TAG=${1:-b1}
timeout 1500 python -m pytest tests/test_gpu_bootstrap.py tests/test_gpu_pipeline.py -m gpu -x -q -s > gpurun_out/boot_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/boot_$TAG.log
tail -30 gpurun_out/boot_$TAG.log
