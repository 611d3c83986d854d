#!/bin/bash
# first GPU validation pass: smoke, kernel/layer parity, quick perf probe
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py -q --maxfail=30 -p no:cacheprovider > gpurun_out/t_kernels.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_lasp2.py -q --maxfail=30 -p no:cacheprovider > gpurun_out/t_lasp2.log 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_cp.py -q --maxfail=30 -p no:cacheprovider > gpurun_out/t_cp.log 2>&1
timeout -s KILL 300 python tools/perf_probe.py 524288 > gpurun_out/perf.log 2>&1
tail -3 gpurun_out/t_*.log
