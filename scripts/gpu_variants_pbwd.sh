#!/bin/bash
# time preprocess_backward for each library variant in libvariants/, both row-reduction kernels
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/base.so
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  for rr in 0 1; do
    echo "== $f RR_PER_THREAD=$rr" >> gpurun_out/variants.log
    VEGS_RR_PER_THREAD=$rr timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep preprocess_backward >> gpurun_out/variants.log
  done
done
cp /tmp/base.so paper_2504_13339_b200/lib/libvegsplat_b200.so
echo "== f64 chain" >> gpurun_out/variants.log
VEGS_BWD_CHAIN_F64=1 VEGS_RR_PER_THREAD=1 timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep preprocess_backward >> gpurun_out/variants.log
