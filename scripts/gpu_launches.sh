#!/bin/bash
# GPU box: ncu launch list (per-kernel durations) of one c2 training step.
mkdir -p gpurun_out
timeout 600 python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_launch.log
