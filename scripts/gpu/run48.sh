mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/pytest_k2_48.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm_48.csv python scripts/profile_step.py --steps 1 --what step > gpurun_out/ncu48.out 2>&1
