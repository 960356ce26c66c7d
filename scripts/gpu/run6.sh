python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu_6.log
timeout 600 python scripts/quick_perf.py lora > gpurun_out/lora_perf_6.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_6.json 2> gpurun_out/bench_6.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_6.csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu_6.out 2>&1
