#!/bin/bash
# time the preprocess stages for each library variant in libvariants/
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/base.so
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $f" >> gpurun_out/variants.log
  timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep preprocess_ >> gpurun_out/variants.log
done
cp /tmp/base.so paper_2504_13339_b200/lib/libvegsplat_b200.so
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
