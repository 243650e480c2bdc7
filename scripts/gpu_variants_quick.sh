#!/bin/bash
# GPU box: kernel timings (scripts/time_kernels.py, channel count $CH, default 3) for each
# libvariants/*.so, run twice in alternating order to expose drift.
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/lib_main.so
: > gpurun_out/variants.log
for pass in 1 2; do
  for f in libvariants/*.so; do
    cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
    echo "== $f (pass $pass)" >> gpurun_out/variants.log
    timeout 300 python scripts/time_kernels.py ${REPS:-10} ${CH:-3} >> gpurun_out/variants.log 2>&1
  done
done
cp /tmp/lib_main.so paper_2504_13339_b200/lib/libvegsplat_b200.so
grep -E "==|composite" gpurun_out/variants.log
