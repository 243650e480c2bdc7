#!/bin/bash
# GPU box: shared projection for TF sweeps -- tests, then the config-3 sweep A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_host.py -q -p no:cacheprovider -x > gpurun_out/proj_tests.log 2>&1
echo "rc=$?" >> gpurun_out/proj_tests.log
for v in "" "--no-shared-projection" "" "--no-shared-projection"; do
  echo "== $v" >> gpurun_out/proj_bench.log
  timeout 900 python bench.py --steps 5 --warmup 3 --no-api --no-cpu-baseline --no-c4 $v 2>&1 | tail -1 > /tmp/b.json
  python - >> gpurun_out/proj_bench.log <<'PY'
import json
d = json.load(open("/tmp/b.json"))
print(round(d["value"], 3), round(d["render_mpx_s"], 1), round(d["render_sweep_c3"]["mpx_s"], 1), d["render_sweep_c3"]["ms_per_render"])
PY
done
