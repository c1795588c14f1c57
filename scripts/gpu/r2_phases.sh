mkdir -p gpurun_out
HE_SM100_LIB=$PWD/build_variants/libhe_phases.so timeout 600 python scripts/role_convtc.py 2>&1 | grep "conv" | tee gpurun_out/phases.log
