#!/bin/bash
# GPU box: launch list of one c2 step, then a full ncu capture of the compositing kernels.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 $NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_launch.log
timeout 600 python scripts/profile_step.py --views 1 > gpurun_out/prof_plain1.log 2>&1 && \
timeout 1500 $NCU --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:composite -c 2 -o gpurun_out/prof_composite python scripts/profile_step.py --views 1 \
    > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
