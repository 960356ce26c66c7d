mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_caas_multiproc_gpu.py tests/test_caas_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_caas_57.log
SDB_SHARE_ONE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 2 --warmup 1 > gpurun_out/bench_n4_57.json 2> gpurun_out/bench_n4_57.err
