#!/bin/bash
# ncu --set full of the three causal-family launches of one cfg3 masked step (fwd, dQ, dK/dV)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:causal_chunk -c 3 \
  -o gpurun_out/r1b_cfg3_causal -f python tools/step_probe.py 524288 1 > gpurun_out/ncu_cfg3.log 2>&1
tail -3 gpurun_out/ncu_cfg3.log
ls -la gpurun_out/
