# probe of a preferred shared-memory carveout for every sdb kernel (SDB_CARVEOUT, a probe build of
# common.cuh launch_k; not in the product): no change, see DESIGN.md section 3
for c in -1 100; do echo "== SDB_CARVEOUT=$c"; SDB_CARVEOUT=$c python scripts/gn_stream_probe.py 2,320,128,128 2,640,64,64 2,1280,32,32 2>&1 | grep -v Warn | cut -c1-200; done > gpurun_out/carveout.log
for c in -1 100; do SDB_CARVEOUT=$c python bench.py --steps 6 --warmup 3 --no-cpu > gpurun_out/carve_$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/carve_$c.json'));print('carveout $c', d['value'], d['caas_accounting']['per_step'])" >> gpurun_out/carveout.log; done
cat gpurun_out/carveout.log
