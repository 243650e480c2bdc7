#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for l in 2 3 4 6 8; do
  echo "== lanes $l" >> gpurun_out/lanes.log
  timeout 300 python bench.py --steps 10 --warmup 3 --lanes $l --no-cpu-baseline --no-sweep --no-c4 --no-api 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print(round(d['value'],3), round(d['e2e']['value'],3), round(d['ms_per_step'],2))" >> gpurun_out/lanes.log
done
done
