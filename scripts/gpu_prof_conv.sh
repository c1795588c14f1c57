# ncu --set full of one conv kernel in scripts/time_convsq.py
#   bash scripts/gpu_prof_conv.sh TAG SKIP   (SKIP 0: conv1 tile, 4: conv2 carry)
mkdir -p gpurun_out
TAG=${1:-cur}
SKIP=${2:-4}
timeout 900 ncu --set full --clock-control none -k regex:k_conv_sqsum --launch-skip $SKIP -c 1 \
   -o gpurun_out/prof_conv_${TAG}_s$SKIP -f python scripts/time_convsq.py 1 > gpurun_out/ncu_conv.log 2>&1
tail -1 gpurun_out/ncu_conv.log; ls -la gpurun_out
