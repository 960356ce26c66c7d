mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_k2_61.log
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu_61.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_61.json 2> gpurun_out/bench_61.err
