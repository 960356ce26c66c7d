mkdir -p gpurun_out
python scripts/xattn_probe.py > gpurun_out/xattn_33.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm_33.csv python scripts/profile_step.py --steps 1 --what step > gpurun_out/ncu33.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"cross_attn" -s 2 -c 2 -o gpurun_out/k7_33 python scripts/xattn_probe.py > gpurun_out/ncu33b.out 2>&1
