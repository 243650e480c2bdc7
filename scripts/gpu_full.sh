#!/bin/bash
# GPU box: full GPU test suite, kernel timings, one bench line (default args unless BENCH_ARGS)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python scripts/time_kernels.py 10 3 > gpurun_out/tk.log 2>&1
timeout 1200 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
