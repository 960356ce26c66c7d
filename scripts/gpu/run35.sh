mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"cross_attn" -s 2 -c 1 -o gpurun_out/k7_35 python scripts/xattn_probe.py > gpurun_out/ncu35.out 2>&1
