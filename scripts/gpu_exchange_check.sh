#!/bin/bash
# GPU box: the bucketed gradient exchange -- NCCL group of one, two gloo ranks on the one
# GPU (pytest), the whole GPU suite, then the N=2 bench path with gloo (timings meaningless)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -p no:cacheprovider \
    -k "multirank or two_rank or nccl" > gpurun_out/exchange_tests.log 2>&1
echo "rc=$?" >> gpurun_out/exchange_tests.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --backend gloo --no-cpu-baseline --no-api \
    > gpurun_out/dp2_gloo.log 2>&1
echo "rc=$?" >> gpurun_out/dp2_gloo.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-api --no-sweep --no-c4 > gpurun_out/bench_quick.log 2>&1
echo "rc=$?" >> gpurun_out/bench_quick.log
