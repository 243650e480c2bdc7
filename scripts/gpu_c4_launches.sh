#!/bin/bash
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file /tmp/c4l.csv python scripts/profile_c4.py --graphs > gpurun_out/c4l.log 2>&1
echo "rc=$?" >> gpurun_out/c4l.log
python scripts/launch_summary.py /tmp/c4l.csv > gpurun_out/c4_launches_summary.txt 2>&1
