mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_convtc.py -x -q > gpurun_out/convtc.log 2>&1; echo "exit $?" >> gpurun_out/convtc.log
tail -2 gpurun_out/convtc.log
timeout 600 python scripts/time_convtc.py 3 > gpurun_out/time_convtc4.log 2>&1; echo "exit $?" >> gpurun_out/time_convtc4.log
head -2 gpurun_out/time_convtc4.log
timeout 300 python scripts/prof_convtc.py conv1 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_convtc -s 1 -c 1 -o gpurun_out/prof_convtc3 python scripts/prof_convtc.py conv1 2 > gpurun_out/ncu3.log 2>&1
tail -1 gpurun_out/ncu3.log
