mkdir -p gpurun_out
cp paper_2407_02031_b200/libsdb.so /tmp/new.so
cp libsdb_old.so paper_2407_02031_b200/libsdb.so
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"layernorm" --csv --log-file gpurun_out/ln_69_old.csv python scripts/ln_probe.py > /dev/null 2>&1
cp /tmp/new.so paper_2407_02031_b200/libsdb.so
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"layernorm" --csv --log-file gpurun_out/ln_69_new.csv python scripts/ln_probe.py > /dev/null 2>&1
