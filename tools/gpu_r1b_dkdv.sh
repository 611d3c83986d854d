#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lasp2.py -q -x -p no:cacheprovider > gpurun_out/t_dkdv.log 2>&1; echo "rc=$?" >> gpurun_out/t_dkdv.log
tail -4 gpurun_out/t_dkdv.log
timeout -s KILL 300 python tools/step_probe.py 524288 1 > gpurun_out/step_dkdv.log 2>&1
cat gpurun_out/step_dkdv.log
LASP2_TRACE=1 python -m paper_2502_07563_b200.build > gpurun_out/build_trace.log 2>&1
timeout -s KILL 300 python tools/trace_dkdv.py 2>&1 | head -20
