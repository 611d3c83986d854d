#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
LASP2_TRACE=1 python -m paper_2502_07563_b200.build > gpurun_out/build_trace.log 2>&1
timeout -s KILL 300 python tools/trace_dkdv.py > gpurun_out/trace_dkdv.log 2>&1
timeout -s KILL 300 python tools/trace_probe.py > gpurun_out/trace_causal.log 2>&1
cat gpurun_out/trace_dkdv.log; head -3 gpurun_out/trace_causal.log
