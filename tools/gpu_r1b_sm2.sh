#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_softmax_kernels.py tests/test_gpu_cp.py tests/test_gpu_hybrid.py -q -x -p no:cacheprovider > gpurun_out/t_sm2.log 2>&1; echo "rc=$?" >> gpurun_out/t_sm2.log
tail -25 gpurun_out/t_sm2.log
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 2>&1 | tail -2
LASP2_SOFTMAX_BWD1=1 timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 2>&1 | tail -1
