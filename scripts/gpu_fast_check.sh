# GPU box: fast-T forward checks and timings (exact vs fast vs fast without fix-up)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -q -p no:cacheprovider > gpurun_out/scale_tests.log 2>&1
echo "rc=$?" >> gpurun_out/scale_tests.log
timeout 300 python scripts/time_kernels.py 10 3 > gpurun_out/tk_exact.log 2>&1
timeout 300 python scripts/time_kernels.py 10 3 fast > gpurun_out/tk_fast.log 2>&1
VEGS_FAST_T_NO_FIXUP=1 timeout 300 python scripts/time_kernels.py 10 3 fast > gpurun_out/tk_fast_nofix.log 2>&1
