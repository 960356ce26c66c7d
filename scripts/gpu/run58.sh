mkdir -p gpurun_out
SDB_SHARE_ONE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 2 --warmup 1 > gpurun_out/bench_n4_58.json 2> gpurun_out/bench_n4_58.err
SDB_SHARE_ONE_GPU=1 SDB_CAAS_TRANSPORT=nccl timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_n2_58.json 2> gpurun_out/bench_n2_58.err
