#!/bin/bash
# GPU box: two-level placement -- binning tests, parity subset, launch lists and bench A/B
# against the single-level placement (VEGS_PLACE_FLAT=1, same library), alternating
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_binning_primitives.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/p2_tests.log 2>&1
echo "rc=$?" >> gpurun_out/p2_tests.log
for flat in 0 1; do
  for cfg in c2 c3; do
    VEGS_PLACE_FLAT=$flat timeout 600 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv python scripts/profile_render.py --config $cfg > gpurun_out/p2_${cfg}_$flat.csv 2>&1
  done
done
for v in "VEGS_X=0" "VEGS_PLACE_FLAT=1" "VEGS_X=0" "VEGS_PLACE_FLAT=1"; do
  echo "== $v" >> gpurun_out/p2_bench.log
  env $v timeout 900 python bench.py --steps 20 --warmup 5 --no-api --no-cpu-baseline 2>&1 | tail -1 > /tmp/b.json
  python - >> gpurun_out/p2_bench.log <<'PY'
import json
d = json.load(open("/tmp/b.json"))
print(round(d["value"], 3), round(d["e2e"]["value"], 3), round(d["render_mpx_s"], 1),
      round(d["render_sweep_c3"]["mpx_s"], 1), round(d["train_densify_c4"]["steps_per_s"], 2),
      {k: round(v["avg_ms"], 4) for k, v in d["stages"].items() if "bin" in k})
PY
done
