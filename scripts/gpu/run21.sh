# K2 v3 (bulk-copied chunks, epoch-recycled fp64 banks): parity, ncu, bench
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/pytest_gpu_21.log
timeout 600 ncu --set full --clock-control none -k regex:"gn_|add_layernorm|geglu" -s 4 -c 4 -o gpurun_out/k2_full_21 python scripts/k2_probe.py > gpurun_out/ncu_21.out 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_21.json 2> gpurun_out/bench_21.err
