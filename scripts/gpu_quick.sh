mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.log 2>&1; echo "ref exit $?" >> gpurun_out/ref.log
tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/ref.log | cut -c1-700
