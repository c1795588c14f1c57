mkdir -p gpurun_out
for e in 0 1 2; do CONVTC_EXP=$e timeout 300 python scripts/role_convtc.py > gpurun_out/role_exp$e.log 2>&1; echo "exp $e"; grep planar gpurun_out/role_exp$e.log; done
