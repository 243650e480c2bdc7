#!/bin/bash
# GPU box (one GPU): the N=2 bench path end to end with the all-reduce on gloo (ranks fold
# onto the one GPU; no kernel waits on another rank), sweep included; timings meaningless.
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --backend gloo --no-cpu-baseline \
    > gpurun_out/dp2_gloo.log 2>&1
echo "rc=$?" >> gpurun_out/dp2_gloo.log
