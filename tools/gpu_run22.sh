#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t22.log 2>&1
tail -3 gpurun_out/t22.log
timeout -s KILL 900 python bench.py > gpurun_out/bench22.json 2> gpurun_out/bench22.err
tail -c 600 gpurun_out/bench22.json
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --eager"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_flat_kernel -s 2 -c 2 -o gpurun_out/b22_cfg2_flat $B --workload cfg2 > gpurun_out/b22_ncu1.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/b22_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | grep b22
