#!/bin/bash
# time the compositing forward for each variant in libvariants/, single-entry vs paired loop
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/base.so
timeout 600 python -m pytest tests/test_gpu_scale.py -q -p no:cacheprovider -k "paired" > gpurun_out/pair_tests.log 2>&1
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  for pr in 0 1; do
    echo "== $f PAIR=$pr" >> gpurun_out/variants.log
    VEGS_FWD_PAIR=$pr timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep composite_forward >> gpurun_out/variants.log
  done
done
cp /tmp/base.so paper_2504_13339_b200/lib/libvegsplat_b200.so
