#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_softmax_kernels.py tests/test_gpu_cp.py -q -p no:cacheprovider -x > gpurun_out/t29.log 2>&1
tail -5 gpurun_out/t29.log
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 > gpurun_out/perf29.log 2>&1

cat gpurun_out/perf29.log
