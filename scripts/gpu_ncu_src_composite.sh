#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/profile_step.py --views 1 > /dev/null 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:composite -c 2 -o /tmp/prof_cs python scripts/profile_step.py --views 1 > gpurun_out/ncu_cs.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_cs.log
/usr/local/cuda/bin/ncu -i /tmp/prof_cs.ncu-rep --page source --csv -k regex:composite_fwd2 > gpurun_out/ncu_src_fwd.csv 2>&1
/usr/local/cuda/bin/ncu -i /tmp/prof_cs.ncu-rep --page source --csv -k regex:composite_bwd4 > gpurun_out/ncu_src_bwd.csv 2>&1
/usr/local/cuda/bin/ncu -i /tmp/prof_cs.ncu-rep --page details --csv > gpurun_out/ncu_cs_details.csv 2>&1
