mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python scripts/bench_primitives.py > gpurun_out/prims.log 2>&1
tail -1 gpurun_out/prims.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_v29.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/bench_v29.log').readline())
print(d['value'], d['step_ms'], d['e2e']['value'], d['e2e']['phase_ms_h2dwait_enc_net_dec'])"
