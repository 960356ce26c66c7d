mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k self_attention 2>&1 | tail -15 > gpurun_out/k8_70.log
timeout 300 python scripts/selfattn_probe.py k8 >> gpurun_out/k8_70.log 2>&1
