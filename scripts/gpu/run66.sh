mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_lora_gpu.py -q -x -k "tma" 2>&1 | tail -2 > gpurun_out/k1_66.log
for na in 2 3 4; do echo "na=$na" >> gpurun_out/k1_66.log; SDB_K1_ASTAGES=$na timeout 300 python scripts/quick_perf.py lora 2 >> gpurun_out/k1_66.log 2>&1; done
