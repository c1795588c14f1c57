mkdir -p gpurun_out
for cfg in "--slab-cap-gb 16" "--slab-cap-gb 4" "--slab-cap-gb 4 --max-outputs 256" "--slab-cap-gb 0"; do
timeout 900 python scripts/run_cfg4.py $cfg > gpurun_out/cfg4_tune.log 2>&1
grep '"config"' gpurun_out/cfg4_tune.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', {k:d[k] for k in ('ms','samples_per_s','max_abs_err_64','peak_hbm_gb_rank0','pool_releases')})" || tail -3 gpurun_out/cfg4_tune.log
done
