mkdir -p gpurun_out
timeout 1200 python scripts/run_cfg4.py --mem-trace > gpurun_out/cfg4_mem.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_mem.log
grep -v "^frame" gpurun_out/cfg4_mem.log | head -60
