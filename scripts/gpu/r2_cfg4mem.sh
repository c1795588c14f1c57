mkdir -p gpurun_out
timeout 2400 python scripts/run_cfg4.py --mem-trace > gpurun_out/cfg4_mem.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_mem.log
grep -v "^frame" gpurun_out/cfg4_mem.log | awk 'NR%8==1' | head -40; tail -c 3000 gpurun_out/cfg4_mem.log
