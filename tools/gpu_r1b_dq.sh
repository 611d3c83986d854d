#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t_dq.log 2>&1; echo "rc=$?" >> gpurun_out/t_dq.log
tail -4 gpurun_out/t_dq.log
timeout -s KILL 300 python tools/step_probe.py 524288 1 > gpurun_out/step_dq.log 2>&1
cat gpurun_out/step_dq.log
