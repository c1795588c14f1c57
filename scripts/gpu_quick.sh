# scratch GPU session (see gpu_round.sh for the full recipe)
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_v18b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv_sqsum<5" -c 1 \
   -o gpurun_out/prof_conv2_v18 -f python scripts/time_convsq.py 1 > gpurun_out/ncu_conv2.log 2>&1
cut -c1-400 gpurun_out/bench_v18b.log; tail -3 gpurun_out/ncu_conv2.log
