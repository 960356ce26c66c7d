mkdir -p gpurun_out
SDB_SHARE_ONE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 3 --steps 2 --warmup 1 > gpurun_out/bench_n3_56.json 2> gpurun_out/bench_n3_56.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/bench_ref_n2_56.json 2> gpurun_out/bench_ref_n2_56.err
