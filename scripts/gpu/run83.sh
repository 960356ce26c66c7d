cp paper_2407_02031_b200/libsdb.so /tmp/libsdb_main.so
for rep in 1 2; do
for v in nr mufu; do
  cp scratch/libsdb_$v.so paper_2407_02031_b200/libsdb.so
  echo "== $v"; timeout 300 python scripts/gn_cluster_probe.py 2>&1 | tail -6 | cut -d'|' -f2
done
done
cp /tmp/libsdb_main.so paper_2407_02031_b200/libsdb.so
