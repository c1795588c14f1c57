# config 4 at full size on one GPU (script, then the layerwise parity test) + tc5 MMA rate probe
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc5.py -q -s -k rate > gpurun_out/tc5rate.log 2>&1
timeout 2400 python scripts/run_cfg4.py > gpurun_out/cfg4_run.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_run.log
grep -v "^frame" gpurun_out/cfg4_run.log | tail -c 1500
timeout 3000 python -m pytest tests/test_gpu_cfg4.py -x -q > gpurun_out/cfg4_full.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_full.log
grep tcgen05 gpurun_out/tc5rate.log; tail -30 gpurun_out/cfg4_full.log
