mkdir -p gpurun_out
timeout 600 python scripts/time_convtc.py 3 > gpurun_out/time_convtc2.log 2>&1; echo "exit $?" >> gpurun_out/time_convtc2.log
cat gpurun_out/time_convtc2.log | tail -6
timeout 300 python scripts/prof_convtc.py conv1 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_convtc -s 1 -c 1 -o gpurun_out/prof_convtc1 python scripts/prof_convtc.py conv1 2 > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
