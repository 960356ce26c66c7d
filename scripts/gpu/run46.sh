mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"gn_" -s 220 -c 2 -o gpurun_out/k2_46 python scripts/k2_launches.py > gpurun_out/ncu46.out 2>&1
