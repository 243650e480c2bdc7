#!/bin/bash
# GPU box: parity tests on the in-tree library, then kernel timings for each libvariants/*.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/lib_main.so
: > gpurun_out/variants.log
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $f" >> gpurun_out/variants.log
  timeout 300 python scripts/time_kernels.py ${REPS:-10} >> gpurun_out/variants.log 2>&1
done
cp /tmp/lib_main.so paper_2504_13339_b200/lib/libvegsplat_b200.so
