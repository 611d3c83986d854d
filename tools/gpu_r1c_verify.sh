#!/bin/bash
# verification after the balanced-LASP-2H / lse-dtype changes: bench line, full GPU suite, smoke
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_gpu_all.log
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 600 python bench.py --workload cfg4 --balanced --no-cpu-baseline > gpurun_out/bench_cfg4_bal.json 2> gpurun_out/bench_cfg4_bal.err
tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/t_gpu_all.log; tail -1 gpurun_out/smoke.log; tail -c 300 gpurun_out/bench_cfg4_bal.json; tail -3 gpurun_out/bench_cfg4_bal.err
