cp paper_2407_02031_b200/libsdb.so /tmp/libsdb_main.so
for v in 256 512; do
  cp scratch/libsdb_$v.so paper_2407_02031_b200/libsdb.so
  echo "== target $v"; timeout 300 python scripts/gn_cluster_probe.py 2>&1 | tail -6
done
cp /tmp/libsdb_main.so paper_2407_02031_b200/libsdb.so
