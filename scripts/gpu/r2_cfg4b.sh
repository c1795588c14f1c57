mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k encrypt > gpurun_out/enc.log 2>&1; tail -1 gpurun_out/enc.log
for mo in 512 256; do
timeout 1200 python scripts/run_cfg4.py --max-outputs $mo > gpurun_out/cfg4_mo$mo.log 2>&1
grep '"config"' gpurun_out/cfg4_mo$mo.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('ms','samples_per_s','peak_hbm_gb_rank0','pool_releases','max_outputs','ms_by_category')})"
done
