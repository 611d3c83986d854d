#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "nomask_local" > gpurun_out/t21a.log 2>&1
tail -3 gpurun_out/t21a.log
timeout -s KILL 300 python tools/flat_probe.py > gpurun_out/flat21.log 2>&1
cat gpurun_out/flat21.log
