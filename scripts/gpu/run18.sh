# the N>1 ControlNet-as-a-service bench path, 3 ranks sharing the one GPU over gloo
SDB_SHARE_ONE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 3 --steps 2 --warmup 1 > gpurun_out/bench_18_caas3.json 2> gpurun_out/bench_18_caas3.err
SDB_SHARE_ONE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 1 --warmup 1 > gpurun_out/bench_18_caas4.json 2> gpurun_out/bench_18_caas4.err
timeout 600 ncu --set full --clock-control none -k regex:"gn_|add_layernorm|geglu" -s 4 -c 4 -o gpurun_out/k2_full_18 python scripts/k2_probe.py > gpurun_out/ncu_18.out 2>&1
timeout 300 python -m pytest tests -q -m gpu -x -k "kernels or pipeline" 2>&1 | tail -3 > gpurun_out/pytest_gpu_18.log
