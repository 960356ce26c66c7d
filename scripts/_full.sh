timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r02_gpu_tests_run4.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_r4.json 2> gpurun_out/bench_r4.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gn_resident -s 2 -c 1 -o gpurun_out/k2r_final python scripts/k2r_ncu.py 2,320,128,128 > gpurun_out/k2r_ncu.log 2>&1
