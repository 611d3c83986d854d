#!/bin/bash
# round-2b evidence (after the dK/dV pair prefetch): bench line + reference arm, launch list, ncu of the
# masked kernels, softmax probe + backward timeline, cfg4 / cfg5 lines, gloo multirank smoke, GPU suite
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
bash tools/gpu.sh bench ref launches
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"causal_chunk" -c 3 \
  -o gpurun_out/r02b_cfg3 -f python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_cfg3.log 2>&1
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 > gpurun_out/perf_softmax.log 2>&1
bash tools/gpu.sh bench:--workload,cfg4,--no-cpu-baseline,--no-secondary bench:--workload,cfg5,--no-cpu-baseline,--no-secondary multirank
cp paper_2502_07563_b200/liblasp2_b200.so /tmp/keep.so
cp ab_so/trace.so paper_2502_07563_b200/liblasp2_b200.so
timeout -s KILL 120 python tools/trace_softmax_bwd.py > gpurun_out/trace_softmax_bwd.log 2>&1
cp /tmp/keep.so paper_2502_07563_b200/liblasp2_b200.so
bash tools/gpu.sh tests smoke
ls -la gpurun_out/*.ncu-rep
