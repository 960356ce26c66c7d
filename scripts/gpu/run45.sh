mkdir -p gpurun_out
for st in 1 4; do for ctas in 2 4; do SDB_GN_STAGES=$st SDB_GN_CTAS=$ctas timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"gn_" --csv --log-file gpurun_out/k2_45_${st}_${ctas}.csv python scripts/k2_launches.py > /dev/null 2>&1; done; done
