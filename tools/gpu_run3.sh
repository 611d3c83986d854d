#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_softmax_kernels.py tests/test_gpu_graph.py tests/test_gpu_cp.py -q --maxfail=30 -p no:cacheprovider > gpurun_out/t3_softmax.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t3_all.log 2>&1
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench3.json 2> gpurun_out/bench3.err
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke3.log 2>&1
tail -5 gpurun_out/t3_*.log
