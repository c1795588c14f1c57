mkdir -p gpurun_out
timeout 600 python scripts/time_convtc.py 3 > gpurun_out/time_convtc.log 2>&1; echo "exit $?" >> gpurun_out/time_convtc.log
cat gpurun_out/time_convtc.log | tail -6
timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_r2c.log 2>&1; echo "exit $?" >> gpurun_out/bench_r2c.log
python -c "
import json;d=json.loads(open('gpurun_out/bench_r2c.log').readline())
print(d['value'], d['step_ms'], d['e2e']['value'], {k:(v['calls'],round(v['ms'],1)) for k,v in d['breakdown'].items()})"
