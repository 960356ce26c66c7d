mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_lora_gpu.py -q -x -k "tma" 2>&1 | tail -3 > gpurun_out/pytest_k1_25.log
timeout 400 python scripts/quick_perf.py lora 2,1 > gpurun_out/k1_sweep_25.log 2>&1
