#!/bin/bash
# compositing forward time for each library variant in libvariants/ (alternating, twice), then
# the parity checks of the forward on the default build
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/base.so
for rep in 1 2; do
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $f" >> gpurun_out/variants.log
  timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep composite_forward >> gpurun_out/variants.log
done
done
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $f" >> gpurun_out/pair_tests.log
  timeout 600 python -m pytest tests/test_gpu_scale.py -q -p no:cacheprovider -k "paired or c2_view_bit" >> gpurun_out/pair_tests.log 2>&1
done
cp /tmp/base.so paper_2504_13339_b200/lib/libvegsplat_b200.so
