#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t13_all.log 2>&1
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench13.json 2> gpurun_out/bench13.err
tail -3 gpurun_out/t13_all.log
