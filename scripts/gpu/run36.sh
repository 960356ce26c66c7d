mkdir -p gpurun_out
for tpw in 1 2 3 4 6; do WARM_ONLY=1 SDB_XATTN_TPW=$tpw python scripts/xattn_probe.py; done > gpurun_out/xattn_36.log 2>&1
