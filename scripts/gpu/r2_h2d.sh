mkdir -p gpurun_out
PYTORCH_CUDA_ALLOC_CONF=backend:cudaMallocAsync timeout 300 python scripts/h2d_probe.py > gpurun_out/h2d_probe.log 2>&1
timeout 300 python scripts/h2d_probe.py >> gpurun_out/h2d_probe.log 2>&1
cat gpurun_out/h2d_probe.log; nvidia-smi -q | grep -i -A3 "compute mode\|copy engine\|async" | head -20
