timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu_14.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_14.json 2> gpurun_out/bench_14.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_14_ref.json 2> gpurun_out/bench_14_ref.err
