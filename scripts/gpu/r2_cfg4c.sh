mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k encrypt > gpurun_out/enc.log 2>&1; tail -1 gpurun_out/enc.log
timeout 900 python -m pytest tests/test_gpu_networks.py -x -q -k cfg4 > gpurun_out/cfg4s.log 2>&1; tail -3 gpurun_out/cfg4s.log
timeout 1200 python scripts/run_cfg4.py > gpurun_out/cfg4_tc.log 2>&1
grep '"config"' gpurun_out/cfg4_tc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('ms','samples_per_s','max_abs_err_64','peak_hbm_gb_rank0','pool_releases','ms_by_category')})" || tail -20 gpurun_out/cfg4_tc.log
timeout 2400 python -m pytest tests/test_gpu_cfg4.py -x -q > gpurun_out/cfg4_full.log 2>&1; tail -15 gpurun_out/cfg4_full.log
