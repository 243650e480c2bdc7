#!/bin/bash
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"place_kernel|block_count|block_place" -c 3 -o /tmp/prof_p2 python scripts/profile_render.py --config c2 > gpurun_out/ncu_p2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_p2.log
python scripts/ncu_summary.py /tmp/prof_p2.ncu-rep > gpurun_out/ncu_p2_summary.txt 2>&1
for k in place_kernel block_count block_place; do
  /usr/local/cuda/bin/ncu -i /tmp/prof_p2.ncu-rep --page source --csv -k regex:$k > gpurun_out/ncu_p2_src_$k.csv 2>&1
done
/usr/local/cuda/bin/ncu -i /tmp/prof_p2.ncu-rep --page raw --csv > gpurun_out/ncu_p2_raw.csv 2>&1
