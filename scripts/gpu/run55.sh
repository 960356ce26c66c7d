mkdir -p gpurun_out
for ab in 1 0 1 0; do SDB_K3_GN_STATS=$ab timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('k3stats=$ab', d['p50_s_per_image'], d['detail']['step_ms_calibrated'], d['clocks']['sm_mhz'])" >> gpurun_out/ab_55.log; done
