mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg2.csv python scripts/bench_primitives.py --cts 256 --reps 1 > gpurun_out/ncu_cfg2.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_cfg2.csv | head -30
