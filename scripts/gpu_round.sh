#!/bin/bash
# GPU box: parity tests, one bench line, then the ncu launch list of one c2 step.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 1200 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
if [ -z "$SKIP_NCU" ]; then
timeout 600 python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_launch.log
fi
