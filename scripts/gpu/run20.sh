# K2 fast paths (branch-free full batches, packed fp32x2): parity, ncu, bench
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/pytest_gpu_20.log
timeout 600 ncu --set full --clock-control none -k regex:"gn_|add_layernorm|geglu" -s 4 -c 4 -o gpurun_out/k2_full_20 python scripts/k2_probe.py > gpurun_out/ncu_20.out 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_20.json 2> gpurun_out/bench_20.err
