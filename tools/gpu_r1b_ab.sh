#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
LASP2_DKDV_DIRECT=1 timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "dkdv or backward_chunk" > gpurun_out/t_ab.log 2>&1; echo "rc=$?" >> gpurun_out/t_ab.log
tail -3 gpurun_out/t_ab.log
timeout -s KILL 300 python tools/step_probe.py 524288 1 2>&1 | tail -2
LASP2_DKDV_DIRECT=1 timeout -s KILL 300 python tools/step_probe.py 524288 1 2>&1 | tail -2
timeout -s KILL 600 python -m pytest tests/test_costmodel.py -q -p no:cacheprovider 2>&1 | tail -2
