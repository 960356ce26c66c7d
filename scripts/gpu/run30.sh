mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu_38.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_38.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_38.json 2> gpurun_out/bench_38.err
