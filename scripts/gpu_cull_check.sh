#!/bin/bash
# GPU box: culled binning -- equivalence tests, then A/B of the bench (step, render, sweep, c4)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -q -p no:cacheprovider -x \
    -k "cull or c3_frame or render_pipeline or trainer or graph" > gpurun_out/cull_tests.log 2>&1
echo "rc=$?" >> gpurun_out/cull_tests.log
for v in "" "--no-cull" "" "--no-cull"; do
  echo "== $v" >> gpurun_out/cull_bench.log
  timeout 900 python bench.py --steps 20 --warmup 5 --no-api --no-cpu-baseline $v 2>&1 | tail -1 > /tmp/b.json
  python - >> gpurun_out/cull_bench.log <<'PY'
import json
d = json.load(open("/tmp/b.json"))
print(round(d["value"], 3), round(d["e2e"]["value"], 3), round(d["render_mpx_s"], 1),
      round(d["render_sweep_c3"]["mpx_s"], 1), round(d["train_densify_c4"]["steps_per_s"], 2),
      {k: round(v["avg_ms"], 4) for k, v in d["stages"].items()})
PY
done
timeout 900 python scripts/time_kernels.py 10 3 > gpurun_out/cull_tk.log 2>&1
