timeout 300 python bench.py --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-250
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-250
