python -m pytest tests -q -m gpu -k "tma or bf16_per_step or batched" 2>&1 | tail -15 > gpurun_out/pytest_gpu_5.log
timeout 600 python scripts/quick_perf.py lora > gpurun_out/lora_perf_5.log 2>&1
