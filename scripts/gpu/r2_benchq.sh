mkdir -p gpurun_out
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-primitives > gpurun_out/benchq.log 2>&1
python - <<'PY'
import json
l=[x for x in open("gpurun_out/benchq.log") if x.startswith("{")][-1]
d=json.loads(l); print(round(d["value"]), round(d["e2e"]["value"]), d["step_ms"], d["e2e"]["phase_ms_h2dwait_enc_net_dec"][:4])
PY
