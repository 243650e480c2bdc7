#!/bin/bash
# GPU box: round-2 profiles -- ncu full capture of the compositing kernels (one c2 view) and of
# the 3M / 1080p config-3 forward, the launch list of one c2 training step and of the bench command.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python scripts/profile_step.py --views 1 > gpurun_out/prof_plain1.log 2>&1 && \
timeout 1500 $NCU --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:composite -c 2 -o gpurun_out/prof_composite_v28 python scripts/profile_step.py --views 1 \
    > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
timeout 600 python scripts/profile_render.py --config c3 > gpurun_out/prof_c3.log 2>&1 && \
timeout 1500 $NCU --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:composite -c 1 -o gpurun_out/prof_c3_fwd_v28 python scripts/profile_render.py --config c3 \
    > gpurun_out/ncu_c3.log 2>&1
echo "c3 rc=$?" >> gpurun_out/ncu_c3.log
timeout 1200 $NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_v28.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_launch.log
timeout 1800 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/bench_cmd_launches_v28.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-api \
    > gpurun_out/ncu_bench.log 2>&1
echo "bench-cmd rc=$?" >> gpurun_out/ncu_bench.log
