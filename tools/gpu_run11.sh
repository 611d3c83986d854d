#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t11_all.log 2>&1
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench11.json 2> gpurun_out/bench11.err
timeout -s KILL 300 python tools/perf_probe.py 524288 > gpurun_out/perf11.log 2>&1
tail -3 gpurun_out/t11_all.log
