#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu_stdout.json 2> gpurun_out/launches.err
for k in tc_causal tc_apply tc_segment; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
     -o gpurun_out/prof_$k python tools/perf_probe.py 524288 > gpurun_out/prof_$k.log 2>&1
done
timeout -s KILL 300 python tools/perf_probe.py 524288 > gpurun_out/perf.log 2>&1
ls -la gpurun_out
