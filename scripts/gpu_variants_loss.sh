#!/bin/bash
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/base.so
for rep in 1 2; do
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $f" >> gpurun_out/variants.log
  timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep -E "loss" >> gpurun_out/variants.log
done
done
cp /tmp/base.so paper_2504_13339_b200/lib/libvegsplat_b200.so
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k "loss or trainer_step or gradient_buffer" > gpurun_out/loss_tests.log 2>&1
