mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k cross 2>&1 | tail -15 > gpurun_out/pytest_k7_60.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"attn" --csv --log-file gpurun_out/k7_60.csv python scripts/xattn_probe.py > /dev/null 2>&1
