mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_networks.py -m gpu -x -q -k "encrypt or decrypt or smoke or cfg1 or encode" > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 300 python scripts/time_encrypt.py 3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_v31.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/bench_v31.log').readline())
print(d['value'], d['step_ms'], d['e2e']['value'], d['e2e']['phase_ms_h2dwait_enc_net_dec'])"
