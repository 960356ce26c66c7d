set -x
python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu_3.log
python bench.py --steps 3 --warmup 2 > gpurun_out/bench_3.json 2> gpurun_out/bench_3.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_3.csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu_3.out 2>&1
nproc > gpurun_out/host_3.txt; free -g >> gpurun_out/host_3.txt; lscpu | head -20 >> gpurun_out/host_3.txt
