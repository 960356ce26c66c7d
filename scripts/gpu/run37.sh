mkdir -p gpurun_out
for tpw in 1 2 3 4; do WARM_ONLY=1 SDB_XATTN_TPW=$tpw timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"cross_attn" --csv --log-file gpurun_out/k7_tpw$tpw.csv python scripts/xattn_probe.py > /dev/null 2>&1; done
