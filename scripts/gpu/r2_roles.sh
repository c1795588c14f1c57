mkdir -p gpurun_out
timeout 600 python scripts/role_convtc.py > gpurun_out/role_convtc.log 2>&1; echo "exit $?" >> gpurun_out/role_convtc.log
bash scripts/gpu/r2_ncu_convtc.sh
cat gpurun_out/role_convtc.log
