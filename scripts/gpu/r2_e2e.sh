mkdir -p gpurun_out
for m in network; do
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-primitives --h2d-overlap $m > gpurun_out/bench_h2d_$m.log 2>&1
python - "$m" <<'PY'
import json,sys
m=sys.argv[1]
l=[x for x in open(f"gpurun_out/bench_h2d_{m}.log") if x.startswith("{")][-1]
d=json.loads(l); print(m, round(d["value"]), round(d["e2e"]["value"]), d["e2e"]["phase_ms_h2dwait_enc_net_dec"])
PY
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plainops.py -x -q > gpurun_out/parity_stage.log 2>&1; tail -2 gpurun_out/parity_stage.log
