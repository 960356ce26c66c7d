mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_caas_multiproc_gpu.py tests/test_caas_gpu.py tests/test_pipeline_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_caas_62.log
SDB_SHARE_ONE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 3 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_n3_62.json 2> gpurun_out/bench_n3_62.err
