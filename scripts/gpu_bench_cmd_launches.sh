#!/bin/bash
# GPU box: binning primitive tests, then the ncu launch list of a shortened bench command
# (every pass of bench.py, fewer repetitions) -- shares only, per-launch times cold-cache
mkdir -p gpurun_out
V=${V:-v31}
timeout 900 python -m pytest tests/test_gpu_binning_primitives.py -q -p no:cacheprovider > gpurun_out/binprim_tests.log 2>&1
echo "rc=$?" >> gpurun_out/binprim_tests.log
timeout 3000 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file /tmp/bench_cmd_launches_$V.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-api \
    --c4-steps 2 --sweep-frames 1 --render-frames 1 > gpurun_out/ncu_bench.log 2>&1
echo "bench-cmd rc=$?" >> gpurun_out/ncu_bench.log
python scripts/launch_summary.py /tmp/bench_cmd_launches_$V.csv > gpurun_out/bench_cmd_launches_${V}_summary.txt 2>&1
gzip -c /tmp/bench_cmd_launches_$V.csv > gpurun_out/bench_cmd_launches_$V.csv.gz
