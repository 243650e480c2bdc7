#!/bin/bash
# GPU box: launch list (kernel durations) of one c3 render (3M Gaussians, 1080p)
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv python scripts/profile_render.py --config c3 > gpurun_out/c3_launches.csv 2>&1
timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv python scripts/profile_render.py --config c2 > gpurun_out/c2r_launches.csv 2>&1
