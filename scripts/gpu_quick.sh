mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_networks.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_v25.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/bench_v25.log').readline())
print(d['value'], d['step_ms'], d['e2e']['value'], d['e2e']['phase_ms_h2dwait_enc_net_dec'], d['clocks'], d['cpu_baseline'])"
