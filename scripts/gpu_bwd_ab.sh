#!/bin/bash
# GPU box: backward A/B (libvariants/new.so vs old.so): parity on new, kernel timings, bench, alternating
mkdir -p gpurun_out
cp paper_2504_13339_b200/lib/libvegsplat_b200.so /tmp/cur.so
cp libvariants/new.so paper_2504_13339_b200/lib/libvegsplat_b200.so
timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/bwdab_tests.log 2>&1
echo "rc=$?" >> gpurun_out/bwdab_tests.log
for rep in 1 2; do
for lib in new old; do
  cp libvariants/$lib.so paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $lib" >> gpurun_out/bwdab_tk.log
  timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep composite_backward >> gpurun_out/bwdab_tk.log
  timeout 300 python scripts/time_kernels.py 10 11 2>&1 | grep composite_backward | sed 's/^/aux /' >> gpurun_out/bwdab_tk.log
done
done
for lib in new old new old; do
  cp libvariants/$lib.so paper_2504_13339_b200/lib/libvegsplat_b200.so
  echo "== $lib" >> gpurun_out/bwdab_bench.log
  timeout 900 python bench.py --steps 20 --warmup 5 --no-api --no-cpu-baseline --no-sweep --no-c4 2>&1 | tail -1 > /tmp/b.json
  python - >> gpurun_out/bwdab_bench.log <<'PY'
import json
d = json.load(open("/tmp/b.json"))
print(round(d["value"], 3), round(d["e2e"]["value"], 3), round(d["render_mpx_s"], 1), {k: round(v["avg_ms"], 4) for k, v in d["stages"].items() if "composite" in k})
PY
done
cp /tmp/cur.so paper_2504_13339_b200/lib/libvegsplat_b200.so
