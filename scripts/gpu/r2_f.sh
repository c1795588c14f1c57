mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc5.py -q -s -k "tmem_read" > gpurun_out/tmemrate.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_wire.py -x -q > gpurun_out/fnew.log 2>&1; echo "exit $?" >> gpurun_out/fnew.log
grep "TMEM" gpurun_out/tmemrate.log; tail -30 gpurun_out/fnew.log
