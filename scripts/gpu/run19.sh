# K2 / K5 / K6 instruction diet + K3 for the UNet's residual adds: parity, ncu, bench
timeout 400 python -m pytest tests -q -m gpu -x -k "kernels or pipeline or caas" 2>&1 | tail -5 > gpurun_out/pytest_gpu_19.log
timeout 600 ncu --set full --clock-control none -k regex:"gn_|add_layernorm|geglu" -s 4 -c 4 -o gpurun_out/k2_full_19 python scripts/k2_probe.py > gpurun_out/ncu_19.out 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_19.json 2> gpurun_out/bench_19.err
