#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python tools/host_probe.py > gpurun_out/host24.log 2>&1
cat gpurun_out/host24.log
