mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/pytest_gpu_27.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_27.json 2> gpurun_out/bench_27.err
