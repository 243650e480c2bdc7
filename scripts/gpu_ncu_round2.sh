#!/bin/bash
# GPU box: one full ncu capture (source-level) of every hot kernel of one c2 view.
mkdir -p gpurun_out
timeout 600 python scripts/profile_step.py --views 1 > gpurun_out/prof_plain1.log 2>&1 && \
timeout 2400 /usr/local/cuda/bin/ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:composite_fwd2_kernel|composite_bwd4|reduce_rows|preprocess_bwd|preprocess_fwd|place_kernel|ssim|adam" \
    -c 12 -o gpurun_out/prof_r2_all python scripts/profile_step.py --views 1 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
