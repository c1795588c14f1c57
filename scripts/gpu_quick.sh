mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "conv_square_sum" > gpurun_out/t.log 2>&1; echo "exit $?" >> gpurun_out/t.log
grep -E "passed|failed|exit" gpurun_out/t.log | tail -2
timeout 300 python scripts/time_convsq.py 3 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_v37.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/bench_v37.log').readline())
print(d['value'], d['step_ms'], d['e2e']['value'])"
