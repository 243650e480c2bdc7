#!/bin/bash
# loss stage (c2) and the config-4 step for each variant in libvariants/
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/base.so
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $f" >> gpurun_out/variants.log
  timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep -E "loss" >> gpurun_out/variants.log
  timeout 600 python scripts/c4_graph_diag.py 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/variants.log
  timeout 300 python -m pytest tests -q -m gpu -p no:cacheprovider -k "loss" >> gpurun_out/variants.log 2>&1
done
cp /tmp/base.so paper_2504_13339_b200/lib/libvegsplat_b200.so
