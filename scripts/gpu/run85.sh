mkdir -p gpurun_out
python bench.py > gpurun_out/bench_85.json 2> gpurun_out/bench_85.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm_85.csv python scripts/profile_step.py --steps 1 --what all > gpurun_out/ncu85a.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"conv_out" -c 1 -o gpurun_out/k9_85 python scripts/convout_probe.py > gpurun_out/ncu85b.out 2>&1
