# K1 CTA-pair kernel: parity + rank sweep (both kernels)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_lora_gpu.py -q -x -k "tma" 2>&1 | tail -15 > gpurun_out/pytest_k1_23.log
timeout 400 python scripts/quick_perf.py lora 1,2 > gpurun_out/k1_sweep_23.log 2>&1
