#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python tools/trace_probe.py 524288 > gpurun_out/trace12.log 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_lasp2.py -q -p no:cacheprovider -x -k "fused_backward or bf16_fast" > gpurun_out/t12.log 2>&1
tail -3 gpurun_out/t12.log
