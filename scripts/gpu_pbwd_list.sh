#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python scripts/time_kernels.py 10 3 > gpurun_out/tk.log 2>&1
timeout 900 python scripts/c4_graph_diag.py > gpurun_out/c4diag.log 2>&1
