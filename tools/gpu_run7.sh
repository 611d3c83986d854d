#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t7_all.log 2>&1
timeout -s KILL 300 python tools/perf_probe.py 524288 > gpurun_out/perf7.log 2>&1
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 > gpurun_out/perf7_softmax.log 2>&1
tail -3 gpurun_out/t7_all.log
