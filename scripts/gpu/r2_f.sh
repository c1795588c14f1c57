mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_wire.py "tests/test_gpu_networks.py::test_cbc_conv_forward_hoisted_rotations_cfg1_ring" -x -q > gpurun_out/fnew.log 2>&1; echo "exit $?" >> gpurun_out/fnew.log
tail -30 gpurun_out/fnew.log
