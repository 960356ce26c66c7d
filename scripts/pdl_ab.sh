# A/B of programmatic dependent launch on the headline step (dev aid)
python -m pytest tests/test_kernels_gpu.py tests/test_pipeline_gpu.py -q -x > gpurun_out/pdl_tests.log 2>&1; tail -2 gpurun_out/pdl_tests.log
for p in 1 0 1; do
  SDB_PDL=$p python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/pdl_bench_$p.json 2> gpurun_out/pdl_bench_$p.err
  python -c "import json;d=json.load(open('gpurun_out/pdl_bench_$p.json'));print('PDL=$p', d['value'], d['p50_s_per_image'], d['detail']['step_ms_calibrated'], d['caas_accounting']['per_step'])"
done
python scripts/gn_stream_probe.py 2,320,128,128 2,640,64,64 2,1280,32,32 > gpurun_out/pdl_gn.log 2>&1
SDB_PDL=0 python scripts/gn_stream_probe.py 2,320,128,128 2,640,64,64 2,1280,32,32 >> gpurun_out/pdl_gn.log 2>&1
