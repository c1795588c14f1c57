mkdir -p gpurun_out
TAG=${1:-t1}
for r in boot12 boot16s; do timeout 600 python scripts/time_bootstrap.py $r; done > gpurun_out/boot_time_$TAG.log 2>&1
cat gpurun_out/boot_time_$TAG.log
