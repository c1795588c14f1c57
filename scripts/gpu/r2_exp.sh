mkdir -p gpurun_out
CONVTC_EXP=1 timeout 300 python scripts/role_convtc.py > gpurun_out/role_exp1.log 2>&1
cat gpurun_out/role_exp1.log | grep planar
