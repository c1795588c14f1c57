# tcgen05 conv iteration: bit-exactness, timings, role split
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_convtc.py -x -q > gpurun_out/convtc_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/convtc_$TAG.log
timeout 600 python scripts/time_convtc.py 3 > gpurun_out/time_convtc_$TAG.log 2>&1
timeout 600 python scripts/role_convtc.py > gpurun_out/role_$TAG.log 2>&1
tail -3 gpurun_out/convtc_$TAG.log; cat gpurun_out/time_convtc_$TAG.log gpurun_out/role_$TAG.log
