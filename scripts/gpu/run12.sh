python -m pytest tests -q -m gpu -x -k "lora or tma or pipeline" 2>&1 | tail -5 > gpurun_out/pytest_gpu_12.log
timeout 600 python scripts/quick_perf.py lora > gpurun_out/lora_perf_12.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lora_patch_tma -c 1 -o gpurun_out/k1_full_12 python scripts/profile_step.py --what patch > gpurun_out/ncu_full_12.out 2>&1
