mkdir -p gpurun_out
for k in 1 2 4; do SDB_INJ_CTAS=$k timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"inject" --csv --log-file gpurun_out/inj_52_$k.csv python scripts/inject_probe.py > /dev/null 2>&1; done
