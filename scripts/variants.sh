#!/bin/bash
# Time composite kernels for each library variant in libvariants/ (scratch experiments).
mkdir -p gpurun_out
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $f" >> gpurun_out/variants.log
  timeout 300 python scripts/time_kernels.py 5 >> gpurun_out/variants.log 2>&1
done
