cp paper_2407_02031_b200/libsdb.so /tmp/libsdb_main.so
for v in 1_12 4_16 5_15 6_18 6_24; do
  cp scratch/libsdb_$v.so paper_2407_02031_b200/libsdb.so
  echo "== $v"; python scripts/other_roofline.py 2>/dev/null | grep K7 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['kernel'][:60], round(d['launch_ms']*1000,2),'us', round(d['frac'],3))"
done
cp /tmp/libsdb_main.so paper_2407_02031_b200/libsdb.so
