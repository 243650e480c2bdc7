#!/bin/bash
# GPU box (V=vNN): GPU tests, ncu full captures of the compositing kernels
# (one c2 training view; one 3M / 1080p config-3 render) summarised here, the bench with the
# fresh capture in profiles/, and the launch lists of one training step and of the bench command.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
V=${V:-v32}
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python scripts/profile_step.py --views 1 > gpurun_out/prof_plain1.log 2>&1 && \
timeout 1500 $NCU --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:composite -c 2 -o /tmp/prof_composite_$V python scripts/profile_step.py --views 1 \
    > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
python scripts/ncu_to_profile.py /tmp/prof_composite_$V.ncu-rep --out gpurun_out/ncu_composite_$V.json >> gpurun_out/ncu_full.log 2>&1
python scripts/ncu_summary.py /tmp/prof_composite_$V.ncu-rep > gpurun_out/ncu_composite_${V}_summary.txt 2>&1
timeout 600 python scripts/profile_render.py --config c3 > gpurun_out/prof_c3.log 2>&1 && \
timeout 1500 $NCU --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:composite -c 1 -o /tmp/prof_c3_fwd_$V python scripts/profile_render.py --config c3 \
    > gpurun_out/ncu_c3.log 2>&1
echo "c3 rc=$?" >> gpurun_out/ncu_c3.log
INST=$(grep -o "splats, [0-9]* instances" gpurun_out/prof_c3.log | grep -o "[0-9]*" | head -1)
python scripts/ncu_to_profile.py /tmp/prof_c3_fwd_$V.ncu-rep --out gpurun_out/ncu_composite_$V.json --suffix _c3 \
    --instances $INST --merge >> gpurun_out/ncu_c3.log 2>&1
python scripts/ncu_summary.py /tmp/prof_c3_fwd_$V.ncu-rep > gpurun_out/ncu_c3_forward_${V}_summary.txt 2>&1
cp gpurun_out/ncu_composite_$V.json profiles/ncu_composite.json
timeout 900 python bench.py > gpurun_out/bench_$V.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$V.log
tail -2 gpurun_out/bench_$V.log | head -1 > gpurun_out/bench_$V.json
timeout 1200 $NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file /tmp/launches_$V.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ncu_launch.log
python scripts/launch_summary.py /tmp/launches_$V.csv > gpurun_out/launches_${V}_summary.txt 2>&1
gzip -c /tmp/launches_$V.csv > gpurun_out/launches_$V.csv.gz
timeout 1800 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file /tmp/bench_cmd_launches_$V.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-api --c4-steps 2 --sweep-frames 1 --render-frames 1 \
    > gpurun_out/ncu_bench.log 2>&1
echo "bench-cmd rc=$?" >> gpurun_out/ncu_bench.log
python scripts/launch_summary.py /tmp/bench_cmd_launches_$V.csv > gpurun_out/bench_cmd_launches_${V}_summary.txt 2>&1
gzip -c /tmp/bench_cmd_launches_$V.csv > gpurun_out/bench_cmd_launches_$V.csv.gz
