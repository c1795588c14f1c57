# new parity tests (plain ops, config 4 at full shape) + config-4 full-size run on one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plainops.py -x -q > gpurun_out/plainops.log 2>&1; echo "exit $?" >> gpurun_out/plainops.log
timeout 1500 python -m pytest tests/test_gpu_networks.py -x -q -k cfg4 > gpurun_out/cfg4_small.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_small.log
timeout 1800 python scripts/run_cfg4.py > gpurun_out/cfg4_run.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_run.log
timeout 2400 python -m pytest tests/test_gpu_cfg4.py -x -q > gpurun_out/cfg4_full.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_full.log
tail -5 gpurun_out/plainops.log gpurun_out/cfg4_small.log; tail -c 2000 gpurun_out/cfg4_run.log; tail -30 gpurun_out/cfg4_full.log
