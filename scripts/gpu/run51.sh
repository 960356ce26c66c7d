mkdir -p gpurun_out

timeout 300 ncu --set full --warp-sampling-interval 0 --clock-control none --cache-control none --import-source on -k regex:"inject_gn" -s 20 -c 1 -o gpurun_out/inj_51 python scripts/inject_probe.py > gpurun_out/ncu51.out 2>&1
