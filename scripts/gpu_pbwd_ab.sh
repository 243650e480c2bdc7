#!/bin/bash
# GPU box: preprocess-backward A/B (row reduction: warp vs per-thread; chain: float32 vs float64)
mkdir -p gpurun_out
for v in "" "VEGS_RR_PER_THREAD=1" "VEGS_BWD_CHAIN_F64=1" "VEGS_RR_PER_THREAD=1 VEGS_BWD_CHAIN_F64=1"; do
  echo "== $v" >> gpurun_out/pbwd_ab.log
  env $v timeout 300 python scripts/time_kernels.py 10 3 2>&1 | grep preprocess_backward >> gpurun_out/pbwd_ab.log
done
timeout 600 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
   -k regex:"reduce_rows|preprocess_bwd" --csv python scripts/profile_step.py --views 1 > gpurun_out/pbwd_launch.csv 2>&1
VEGS_RR_PER_THREAD=1 VEGS_BWD_CHAIN_F64=1 timeout 600 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
   -k regex:"reduce_rows|preprocess_bwd" --csv python scripts/profile_step.py --views 1 > gpurun_out/pbwd_launch_old.csv 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
