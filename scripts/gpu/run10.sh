python -m pytest tests -q -m gpu -k "caas or pipeline" 2>&1 | tail -5 > gpurun_out/pytest_gpu_10.log
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --mode branch > gpurun_out/bench_10_branch.json 2> gpurun_out/bench_10_branch.err
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --mode serial > gpurun_out/bench_10_serial.json 2> gpurun_out/bench_10_serial.err
