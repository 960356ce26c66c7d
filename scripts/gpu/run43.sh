mkdir -p gpurun_out
for pdl in 0 1; do SDB_GN_PDL=$pdl timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --cache-control none -k regex:"gn_" --csv --log-file gpurun_out/k2_43_$pdl.csv python scripts/k2_probe.py > /dev/null 2>&1; done
