mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k cross 2>&1 | tail -5 > gpurun_out/pytest_k7_34.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cross_attn|sdpa" --csv --log-file gpurun_out/k7_34.csv python scripts/xattn_probe.py > gpurun_out/ncu34.out 2>&1
