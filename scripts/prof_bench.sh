#!/bin/bash
# Profiling recipe for one bench network pass (run under gpurun from the repo root).
#   1. plain run (must exit 0)   2. launch list   3. ncu --set full of the top kernels
set -e
mkdir -p gpurun_out
TAG=${1:-cur}
python bench.py --profile-steps 1 > gpurun_out/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-steps 1 > gpurun_out/ncu_l_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${2:-k_conv_mma}" -c ${3:-2} \
    -o gpurun_out/prof_$TAG -f python bench.py --profile-steps 1 > gpurun_out/ncu_f_$TAG.log 2>&1
