#!/bin/bash
# GPU box: binning A/B (libvariants/new.so vs base.so): parity subset on new, launch lists, bench x2 alternating
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/cur.so
cp libvariants/new.so paper_2504_13339_b200/lib/libvegsplat_b200.so
timeout 1200 python -m pytest tests/test_gpu_binning_primitives.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/binab_tests.log 2>&1
echo "rc=$?" >> gpurun_out/binab_tests.log
for lib in new base; do
  cp libvariants/$lib.so paper_2504_13339_b200/lib/libvegsplat_b200.so
  for cfg in c2 c3; do
    timeout 600 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv python scripts/profile_render.py --config $cfg > gpurun_out/ab_${cfg}_$lib.csv 2>&1
  done
done
for lib in new base new base; do
  cp libvariants/$lib.so paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $lib" >> gpurun_out/binab_bench.log
  timeout 900 python bench.py --steps 20 --warmup 5 --no-api --no-cpu-baseline 2>&1 | tail -1 > /tmp/b.json
  python - >> gpurun_out/binab_bench.log <<'PY'
import json
d = json.load(open("/tmp/b.json"))
print(round(d["value"], 3), round(d["e2e"]["value"], 3), round(d["render_mpx_s"], 1),
      round(d["render_sweep_c3"]["mpx_s"], 1), round(d["train_densify_c4"]["steps_per_s"], 2),
      {k: round(v["avg_ms"], 4) for k, v in d["stages"].items() if "bin" in k})
PY
done
cp /tmp/cur.so paper_2504_13339_b200/lib/libvegsplat_b200.so
