# A/B the fused-conv variants in build_variants/ (HE_SM100_LIB) against the in-tree library
mkdir -p gpurun_out
TAG=${1:-v}
timeout 900 python -m pytest tests/test_gpu_convtc.py -x -q > gpurun_out/convtc_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/convtc_$TAG.log
tail -3 gpurun_out/convtc_$TAG.log
for v in "" $(ls build_variants/*.so 2>/dev/null); do
  echo "== variant ${v:-in-tree}" >> gpurun_out/role_$TAG.log
  HE_SM100_LIB=${v:+$PWD/$v} timeout 600 python scripts/role_convtc.py >> gpurun_out/role_$TAG.log 2>&1
done
cat gpurun_out/role_$TAG.log
bash scripts/gpu/r2_benchq.sh
