# round-2 validation: full GPU suite, headline bench line, ncu of the streamed K2 form (dev aid)
python -m pytest tests -m gpu -x -q > gpurun_out/v_gputests.log 2>&1; tail -2 gpurun_out/v_gputests.log
python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err
python -c "import json;d=json.load(open('gpurun_out/v_bench.json'));print(d['value'],d['e2e']['value'],d['p50_s_per_image']);[print(k['kernel'][:60],round(k['frac'],3),round(k['launch_ms']*1e3,1)) for k in d['roofline_other_kernels']]"
ncu --set full --import-source on --clock-control none -k regex:gn_stream -c 1 -o gpurun_out/gs64_full python scripts/k2_forms_ncu.py 2,640,64,64 > /dev/null 2>&1
