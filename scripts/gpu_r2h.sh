mkdir -p gpurun_out
timeout 300 python scripts/prof_convtc.py conv2 2 > gpurun_out/prof_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_convtc -s 1 -c 1 -o gpurun_out/prof_convtc_c2 python scripts/prof_convtc.py conv2 2 > gpurun_out/ncu_c2.log 2>&1
tail -1 gpurun_out/ncu_c2.log
