#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:tc_flat_kernel -c 2 \
   -o gpurun_out/r1c_cfg2_flat -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_flat.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"causal_chunk|segment_states" -c 4 \
   -o gpurun_out/r1c_cfg3 -f python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_cfg3.log 2>&1
ls -la gpurun_out/*.ncu-rep
