#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python tools/eager_probe.py > gpurun_out/eager25.log 2>&1

cat gpurun_out/eager25.log
