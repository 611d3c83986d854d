#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python tools/trace_softmax_fwd.py > gpurun_out/trace26.log 2>&1
cat gpurun_out/trace26.log
