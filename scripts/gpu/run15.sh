timeout 900 python -m pytest tests -q -m gpu -x -k "kernels or pipeline or caas_gpu" 2>&1 | tail -6 > gpurun_out/pytest_gpu_15.log
timeout 300 python scripts/gemm_probe.py > gpurun_out/gemm_15.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_15.json 2> gpurun_out/bench_15.err
