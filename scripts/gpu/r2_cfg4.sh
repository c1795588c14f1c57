# config 4 at full size on one GPU (script, then the layerwise parity test) + cfg2 primitives line
mkdir -p gpurun_out
timeout 300 python bench.py --workload cfg2 > gpurun_out/cfg2.log 2>&1; echo "exit $?" >> gpurun_out/cfg2.log
timeout 2400 python scripts/run_cfg4.py > gpurun_out/cfg4_run.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_run.log
grep -v "^frame" gpurun_out/cfg4_run.log | tail -c 3000
timeout 3000 python -m pytest tests/test_gpu_cfg4.py -x -q > gpurun_out/cfg4_full.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_full.log
tail -c 1500 gpurun_out/cfg2.log; tail -30 gpurun_out/cfg4_full.log
