# re-entry check: parity, smoke, bench, warm launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu_22.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_22.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_22.json 2> gpurun_out/bench_22.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_22.json 2> gpurun_out/bench_ref_22.err
