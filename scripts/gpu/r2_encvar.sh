mkdir -p gpurun_out; rm -f gpurun_out/encvar.log
for v in "" $(ls build_variants/libhe_enc_*.so 2>/dev/null); do
  echo "== ${v:-in-tree}" >> gpurun_out/encvar.log
  HE_SM100_LIB=${v:+$PWD/$v} timeout 300 python scripts/time_encrypt.py 5 >> gpurun_out/encvar.log 2>&1
done
cat gpurun_out/encvar.log
