mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"gn_" -s 40 -c 4 -o gpurun_out/k2_41 python scripts/k2_probe.py > gpurun_out/ncu41.out 2>&1
