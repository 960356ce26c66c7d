for d in 0 1 2 3; do echo "== SDB_GN_DBG=$d"; SDB_GN_DBG=$d python scripts/gn_stream_probe.py 2,640,32,32 2,320,128,128 2,640,64,64 2>&1 | grep -v Warn; done
