#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k probe > gpurun_out/t27.log 2>&1
tail -15 gpurun_out/t27.log
