#!/bin/bash
# end-of-session evidence: bench line + reference arm, launch list, cfg5 sweeps, full GPU suite, smoke
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu_stdout.json 2> gpurun_out/launches.err
timeout -s KILL 900 python tools/cfg5_sweep.py > gpurun_out/cfg5_sweep.log 2>&1
timeout -s KILL 300 python tools/cfg5_sweep.py --unmasked 131072 1048576 > gpurun_out/cfg2_w8_sweep.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_gpu_all.log
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -c 300 gpurun_out/bench.json; tail -2 gpurun_out/t_gpu_all.log; tail -1 gpurun_out/smoke.log
