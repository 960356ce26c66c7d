set -x
python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu_4.log
timeout 600 python scripts/quick_perf.py lora > gpurun_out/lora_perf_4.log 2>&1
