#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -q -p no:cacheprovider -k "graph" > gpurun_out/graph_tests.log 2>&1
echo "rc=$?" >> gpurun_out/graph_tests.log
timeout 1200 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err
echo "rc=$?" >> gpurun_out/ref.err
