timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "self_attention" > gpurun_out/fmha_tests.log 2>&1; tail -3 gpurun_out/fmha_tests.log
timeout 120 python scripts/fmha2_probe.py 2>&1 | grep -v Warn > gpurun_out/fmha2_sk.log
cat gpurun_out/fmha2_sk.log
