#!/bin/bash
# step-gap probe: cfg3 masked step eager / graph / kernel-sum, with and without PDL
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
( timeout -s KILL 300 python tools/step_probe.py 524288 1
  LASP2_NO_PDL=1 timeout -s KILL 300 python tools/step_probe.py 524288 1
  timeout -s KILL 300 python tools/step_probe.py 131072 0 ) > gpurun_out/step.log 2>&1
cat gpurun_out/step.log
