mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pipeline_gpu.py tests/test_caas_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_batch_64.log
timeout 1200 python bench.py --steps 3 --warmup 3 --batch 8 --no-cpu > gpurun_out/bench_b8_64.json 2> gpurun_out/bench_b8_64.err
