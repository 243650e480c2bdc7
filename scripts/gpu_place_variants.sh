#!/bin/bash
# GPU box: two-level placement variants in libvariants/: placement tests, kernel times (ncu launch
# lists of one c2 / c3 render), bench lines
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/cur.so
for lib in both b1 t1024; do
  cp libvariants/$lib.so paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $lib" >> gpurun_out/pv_tests.log
  timeout 600 python -m pytest tests/test_gpu_binning_primitives.py -q -p no:cacheprovider -x 2>&1 | tail -1 >> gpurun_out/pv_tests.log
  for cfg in c2 c3; do
    timeout 600 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv python scripts/profile_render.py --config $cfg > gpurun_out/pv_${cfg}_$lib.csv 2>&1
  done
done
for lib in both b1 t1024 both b1 t1024; do
  cp libvariants/$lib.so paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $lib" >> gpurun_out/pv_bench.log
  timeout 900 python bench.py --steps 20 --warmup 5 --no-api --no-cpu-baseline --no-c4 2>&1 | tail -1 > /tmp/b.json
  python - >> gpurun_out/pv_bench.log <<'PY'
import json
d = json.load(open("/tmp/b.json"))
print(round(d["value"], 3), round(d["e2e"]["value"], 3), round(d["render_mpx_s"], 1), round(d["render_sweep_c3"]["mpx_s"], 1))
PY
done
cp /tmp/cur.so paper_2504_13339_b200/lib/libvegsplat_b200.so
