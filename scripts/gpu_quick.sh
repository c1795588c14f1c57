mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_v35.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/bench_v35.log').readline())
print(d['value'], d['step_ms'], d['e2e']['value'], d['e2e']['phase_ms_h2dwait_enc_net_dec'], d['roofline']['frac'])"
