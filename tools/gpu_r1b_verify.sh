#!/bin/bash
# re-entry verification: smoke, full GPU suite, default bench line
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_gpu.log
timeout -s KILL 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout -s KILL 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
tail -3 gpurun_out/smoke.log gpurun_out/t_gpu.log; tail -c 600 gpurun_out/bench.log; tail -c 400 gpurun_out/bench_ref.log
