mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm_59.csv python scripts/profile_step.py --steps 1 --what all > gpurun_out/ncu59a.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"cross_attn" -s 2 -c 1 -o gpurun_out/k7_59 python scripts/xattn_probe.py > gpurun_out/ncu59b.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gn_|inject" -s 60 -c 3 -o gpurun_out/k2_59 python scripts/inject_probe.py > gpurun_out/ncu59c.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gn_stats|gn_apply" -s 40 -c 2 -o gpurun_out/k2b_59 python scripts/k2_probe.py > gpurun_out/ncu59d.out 2>&1
