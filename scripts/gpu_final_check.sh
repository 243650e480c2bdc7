#!/bin/bash
# GPU box: full GPU suite, smoke, the N=2 plumbing run (gloo, ranks folded onto one GPU), one
# reference-arm run and one bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --backend gloo --no-cpu-baseline --no-api \
    --c4-steps 2 > gpurun_out/dp2_gloo.log 2>&1
echo "rc=$?" >> gpurun_out/dp2_gloo.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
