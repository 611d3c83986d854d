#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python tools/trace_softmax.py > gpurun_out/trace17.log 2>&1
timeout -s KILL 300 python tools/trace_probe.py 524288 > gpurun_out/trace17_causal.log 2>&1
