#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t9.log 2>&1
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench9.json 2> gpurun_out/bench9.err
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 > gpurun_out/perf9_softmax.log 2>&1
tail -3 gpurun_out/t9.log
