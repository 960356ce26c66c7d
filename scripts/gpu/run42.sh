mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "groupnorm" 2>&1 | tail -3 > gpurun_out/pytest_k2_42.log
for cfg in "0 2" "1 2" "1 3" "1 4" "1 6"; do set -- $cfg; echo "pdl=$1 ctas=$2" >> gpurun_out/k2_42.log; SDB_GN_PDL=$1 SDB_GN_CTAS=$2 python scripts/other_roofline.py 2>&1 | grep K2 | cut -c1-160 >> gpurun_out/k2_42.log; done
