mkdir -p gpurun_out
SDB_DEBUG=1 timeout 400 python scripts/quick_perf.py lora 2,1 > gpurun_out/k1_sweep_24.log 2>&1
