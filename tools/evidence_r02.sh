#!/bin/bash
# round-2 evidence: bench line + reference arm, launch list, ncu captures, cfg4 line, gloo multirank smoke
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
bash tools/gpu.sh bench ref launches
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"tc_flat_kernel" -c 2 \
  -o gpurun_out/r02_cfg2_flat -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_cfg2.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"causal_chunk|segment_states" -c 4 \
  -o gpurun_out/r02_cfg3 -f python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_cfg3.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"tc_softmax" -c 2 \
  -o gpurun_out/r02_softmax -f python tools/perf_probe.py 0 softmax 32768 > gpurun_out/ncu_softmax.log 2>&1
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 > gpurun_out/perf_softmax.log 2>&1
bash tools/gpu.sh bench:--workload,cfg4,--no-cpu-baseline,--no-secondary multirank
ls -la gpurun_out/*.ncu-rep
