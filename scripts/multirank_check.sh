# N>1 bench control flow on one GPU: 2 ranks, gloo process group, small text per rank
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --bases-per-rank 16000000 --no-cpu-baseline 2>&1 | grep -v Warning | tail -5
