mkdir -p gpurun_out
for sk in 0 500 1000 1800 2500 4000; do
  echo "== skew $sk" >> gpurun_out/skew.log
  CONVTC_SKEW=$sk timeout 600 python scripts/role_convtc.py 2>&1 | sed -E "s/'prod[^}]*'epi wait/'epi wait/" >> gpurun_out/skew.log
done
cat gpurun_out/skew.log
