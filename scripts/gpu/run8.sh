python -m pytest tests -q -m gpu -x 2>&1 | tail -8 > gpurun_out/pytest_gpu_8.log
timeout 600 python scripts/quick_perf.py lora > gpurun_out/lora_perf_8.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_8.json 2> gpurun_out/bench_8.err
