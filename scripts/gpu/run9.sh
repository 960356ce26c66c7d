python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu_9.log
timeout 900 python -m paper_2407_02031_b200.profile > gpurun_out/profile_9.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_9.json 2> gpurun_out/bench_9.err
