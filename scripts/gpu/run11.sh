timeout 900 python -m pytest tests/test_caas_multiproc_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu_11.log
timeout 300 python scripts/attn_probe.py > gpurun_out/attn_11.log 2>&1
