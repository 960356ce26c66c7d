set -x
python scripts/gn_stream_probe.py > gpurun_out/gs_probe.log 2>&1
for sc in 40,8 40,16 80,16 80,8 40,4 160,16; do
  echo "== $sc" >> gpurun_out/gs_sweep.log
  SDB_GN_SLAB=$sc python scripts/gn_stream_probe.py 2,320,128,128 2,640,64,64 16,320,128,128 >> gpurun_out/gs_sweep.log 2>&1
done
python -m pytest tests/test_kernels_gpu.py -q -x -k "groupnorm" > gpurun_out/gs_tests.log 2>&1
tail -3 gpurun_out/gs_tests.log
