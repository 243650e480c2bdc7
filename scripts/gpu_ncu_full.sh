#!/bin/bash
# GPU box: full ncu capture of the two compositing kernels of one 1024^2 view.
mkdir -p gpurun_out
timeout 600 python scripts/profile_step.py --views 1 > gpurun_out/prof_plain1.log 2>&1 && \
timeout 1500 /usr/local/cuda/bin/ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:${NCU_KERNELS:-composite} -c ${NCU_COUNT:-2} -o gpurun_out/${NCU_OUT:-prof_composite} \
    python scripts/profile_step.py --views 1 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
