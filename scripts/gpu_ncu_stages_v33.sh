#!/bin/bash
# GPU box: ncu --set full of the non-compositing kernels of one c2 view (stage bounds);
# the report is summarised on the box (raw-page csv) and not returned (size).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python scripts/profile_step.py --views 1 > gpurun_out/prof_plain1.log 2>&1 && \
timeout 2400 $NCU --profile-from-start off --set full --clock-control none \
    -k "regex:preprocess|reduce_rows|place|chunk|ssim|adam|Onesweep|depth|bin_rect|tile_diff|tile_total|kept_list|tile_group" -c 48 -o /tmp/prof_stages_v33 \
    python scripts/profile_step.py --views 1 > gpurun_out/ncu_stages.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_stages.log
$NCU -i /tmp/prof_stages_v33.ncu-rep --page raw --csv > gpurun_out/stages_raw_v33.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/prof_stages_v33.ncu-rep > gpurun_out/ncu_stages_v33_summary.txt 2>&1

python scripts/stage_bounds.py gpurun_out/stages_raw_v33.csv > gpurun_out/stage_bounds_v33.txt 2>&1
