mkdir -p gpurun_out
timeout 300 python scripts/prof_convtc.py conv1pl 2 > gpurun_out/prof_plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_convtc -s 1 -c 1 -f -o gpurun_out/ncu_conv1pl_s6 python scripts/prof_convtc.py conv1pl 2 > gpurun_out/ncu_c1.log 2>&1
cat gpurun_out/prof_plain1.log; tail -2 gpurun_out/ncu_c1.log
