#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python tools/flat_probe.py > gpurun_out/flat20.log 2>&1
cat gpurun_out/flat20.log
