mkdir -p gpurun_out
for m in 1 2; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"lora_patch_(tma|pair)" -s 1 -c 1 -o gpurun_out/k1_r64_m$m python scripts/k1_probe.py 64 $m > gpurun_out/ncu26_$m.out 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"lora_patch_(tma|pair)" -s 1 -c 1 -o gpurun_out/k1_r232_m2 python scripts/k1_probe.py 8,32,64,128 2 > gpurun_out/ncu26_232.out 2>&1
