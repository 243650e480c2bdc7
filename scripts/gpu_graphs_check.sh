#!/bin/bash
# GPU box: graph-step tests, then a bench line with graphs (default) and one without
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -q -p no:cacheprovider -k "graph" > gpurun_out/graph_tests.log 2>&1
echo "rc=$?" >> gpurun_out/graph_tests.log
timeout 1200 python bench.py --no-cpu-baseline --no-api > gpurun_out/bench_graphs.json 2> gpurun_out/bench_graphs.err
echo "rc=$?" >> gpurun_out/bench_graphs.err
timeout 1200 python bench.py --no-cpu-baseline --no-api --no-sweep --no-graphs > gpurun_out/bench_eager.json 2> gpurun_out/bench_eager.err
echo "rc=$?" >> gpurun_out/bench_eager.err
