for cfg in 512,2 256,4 256,2 512,1 128,8 256,8; do
  echo "== SDB_GN_APPLY=$cfg"; SDB_GN_APPLY=$cfg python scripts/k2_bench.py 2>&1 | grep -v Warn | head -3
done
