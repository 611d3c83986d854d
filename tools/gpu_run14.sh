#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python tools/nscan_probe.py > gpurun_out/nscan14.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --eager"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_fused_apply -s 2 -c 2 -o gpurun_out/b14_cfg2_fused $B --workload cfg2 > gpurun_out/b14_ncu1.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:"tc_segment|tc_apply_state" -s 2 -c 2 -o gpurun_out/b14_cfg2_segapply $B --workload cfg2 > gpurun_out/b14_ncu2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:"tc_causal" -s 3 -c 2 -o gpurun_out/b14_cfg3_causal $B --workload cfg3 > gpurun_out/b14_ncu3.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/b14_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | tail -20
