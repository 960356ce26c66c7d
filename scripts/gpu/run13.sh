timeout 600 python -m pytest tests -q -m gpu -x -k "lora or tma" 2>&1 | tail -5 > gpurun_out/pytest_gpu_13.log
timeout 600 python scripts/quick_perf.py lora > gpurun_out/lora_perf_13.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_13.log 2>&1
timeout 900 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_warm_13.csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu_13.out 2>&1
