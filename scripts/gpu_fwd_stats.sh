#!/bin/bash
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/base.so
cp libvariants/stats.so paper_2504_13339_b200/lib/libvegsplat_b200.so
timeout 600 python scripts/fwd_stats.py c2 > gpurun_out/fwd_stats.log 2>&1
timeout 600 python scripts/fwd_stats.py c3 >> gpurun_out/fwd_stats.log 2>&1
cp /tmp/base.so paper_2504_13339_b200/lib/libvegsplat_b200.so
