timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gn_|add_layernorm|geglu" -s 4 -c 4 -o gpurun_out/k2_full_16 python scripts/k2_probe.py > gpurun_out/ncu_16.out 2>&1
timeout 300 python -m pytest tests -q -m gpu -x -k "kernels" 2>&1 | tail -3 > gpurun_out/pytest_gpu_16.log
