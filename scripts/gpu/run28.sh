mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm_28.csv python scripts/profile_step.py --steps 1 --what all > gpurun_out/ncu28.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lora_patch_pair" -s 1 -c 1 -o gpurun_out/k1_pair_r128_28 python scripts/k1_probe.py 64,64 0 > gpurun_out/ncu28b.out 2>&1
