#!/bin/bash
# full config-2 step time for each library variant in libvariants/ (alternating, twice)
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/base.so
for rep in 1 2; do
for f in libvariants/*.so; do
  cp "$f" paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $f" >> gpurun_out/variants.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweep --no-c4 --no-api 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print(round(d['value'],3), round(d['ms_per_step'],2), {k: round(v['avg_ms'],3) for k,v in d['kernels'].items()})" >> gpurun_out/variants.log
done
done
cp /tmp/base.so paper_2504_13339_b200/lib/libvegsplat_b200.so
