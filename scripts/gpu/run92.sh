mkdir -p gpurun_out
export PYTHONPATH=.
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"conv_out_mma" -c 1 -o gpurun_out/k9_92 python scripts/convout_probe.py > gpurun_out/ncu92a.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gn_cluster" -c 1 -o gpurun_out/gnc_92 python scripts/gn_cluster_one.py > gpurun_out/ncu92b.out 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gn_stats|gn_apply" -s 40 -c 2 -o gpurun_out/k2_92 python scripts/k2_probe.py > gpurun_out/ncu92c.out 2>&1
ls -la gpurun_out/*_92.ncu-rep
