#!/bin/bash
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"place_kernel|chunk_offsets|chunk_count" -c 3 -o /tmp/prof_place python scripts/profile_render.py --config c3 > gpurun_out/ncu_place.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_place.log
python scripts/ncu_summary.py /tmp/prof_place.ncu-rep > gpurun_out/ncu_place_summary.txt 2>&1
/usr/local/cuda/bin/ncu -i /tmp/prof_place.ncu-rep --page source --csv -k regex:place_kernel > gpurun_out/ncu_place_source.csv 2>&1
/usr/local/cuda/bin/ncu -i /tmp/prof_place.ncu-rep --page details --csv -k regex:place_kernel > gpurun_out/ncu_place_details.csv 2>&1
