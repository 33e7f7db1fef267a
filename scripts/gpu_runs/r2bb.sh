#!/bin/bash
# round 2: N>1 bench path on the final code (two ranks on one GPU via
# LKV_BENCH_ONE_GPU: fused gather verified against NCCL on the first step)
O=gpurun_out; mkdir -p $O
LKV_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29537 bench.py --gpus 2 --steps 2 --warmup 3 --no-rows --no-cpu-baseline > $O/r2bb_bench_2r1g.json 2> $O/r2bb_bench_2r1g.err; echo "2r1g rc=$?"
