mkdir -p gpurun_out
timeout 300 python scripts/prof_convtc.py conv2pl 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_convtc -s 1 -c 1 -f -o gpurun_out/ncu_conv2pl_s6 python scripts/prof_convtc.py conv2pl 2 > gpurun_out/ncu_c2.log 2>&1
cat gpurun_out/prof_plain.log; tail -2 gpurun_out/ncu_c2.log
