timeout 600 ncu --set full --clock-control none -k regex:"gn_|add_layernorm|geglu" -s 4 -c 4 -o gpurun_out/k2_full_17 python scripts/k2_probe.py > gpurun_out/ncu_17.out 2>&1
timeout 300 python -m pytest tests -q -m gpu -x -k "kernels or pipeline" 2>&1 | tail -3 > gpurun_out/pytest_gpu_17.log
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_17.json 2> gpurun_out/bench_17.err
