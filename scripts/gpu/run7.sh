python -m pytest tests -q -m gpu -x -k "lora or tma" 2>&1 | tail -5 > gpurun_out/pytest_gpu_7.log
timeout 600 python scripts/quick_perf.py lora > gpurun_out/lora_perf_7.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:lora_patch_tma -c 1 -o gpurun_out/k1_full_7 python scripts/profile_step.py --what patch > gpurun_out/ncu_full_7.out 2>&1
ncu --set full --clock-control none -k regex:"gn_stats|gn_apply|add_layernorm|geglu|residual_inject" -c 8 -o gpurun_out/small_full_7 python scripts/profile_step.py --what step > gpurun_out/ncu_small_7.out 2>&1
