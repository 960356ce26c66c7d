mkdir -p gpurun_out
for pr in 3 0; do for k in 2 8; do SDB_INJ_PROBE=$pr SDB_INJ_CTAS=$k timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"inject" --csv --log-file gpurun_out/inj_53_${pr}_$k.csv python scripts/inject_probe.py > /dev/null 2>&1; done; done
