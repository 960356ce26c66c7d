timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "self_attention" > gpurun_out/fmha_tests.log 2>&1; tail -3 gpurun_out/fmha_tests.log
for bk in 32 64; do echo "== SDB_FMHA_BK=$bk"; SDB_FMHA_BK=$bk timeout 120 python scripts/fmha2_probe.py 2>&1 | grep -v Warn; done > gpurun_out/fmha2_bk.log
cat gpurun_out/fmha2_bk.log
