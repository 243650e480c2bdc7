#!/bin/bash
# binning stage time for each library variant in libvariants/ (alternating, twice)
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/base.so
for rep in 1 2; do
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $f" >> gpurun_out/variants.log
  timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep -E "bin_sort|adam" >> gpurun_out/variants.log
done
done
cp /tmp/base.so paper_2504_13339_b200/lib/libvegsplat_b200.so
