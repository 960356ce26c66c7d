mkdir -p gpurun_out
SDB_GN_DIRECT=1 timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "groupnorm or inject" 2>&1 | tail -2 > gpurun_out/k2_73.log
for d in 0 1; do SDB_GN_DIRECT=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"gn_" --csv --log-file gpurun_out/k2_73_$d.csv python scripts/k2_launches.py > /dev/null 2>&1; SDB_GN_DIRECT=$d python scripts/other_roofline.py 2>&1 | grep K2 | cut -c1-120 >> gpurun_out/k2_73.log; done
