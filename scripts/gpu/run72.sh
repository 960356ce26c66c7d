mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "groupnorm or inject" 2>&1 | tail -2 > gpurun_out/k2_72.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"gn_" --csv --log-file gpurun_out/k2_72.csv python scripts/k2_launches.py > /dev/null 2>&1
python scripts/other_roofline.py 2>&1 | grep K2 | cut -c1-150 >> gpurun_out/k2_72.log
