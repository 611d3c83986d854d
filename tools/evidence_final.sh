#!/bin/bash
# final round-2 evidence: bench line + reference arm, launch list, ncu of the masked + flat kernels, cfg4 /
# cfg5 lines, rank probes at the W=8 shapes, gloo multirank smoke, GPU suite, smoke
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
bash tools/gpu.sh bench ref launches
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"causal_chunk|segment_states" -c 4 \
  -o gpurun_out/fin_cfg3 -f python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_cfg3.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"tc_flat_kernel" -c 2 \
  -o gpurun_out/fin_cfg2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_cfg2.log 2>&1
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 > gpurun_out/perf_softmax.log 2>&1
bash tools/gpu.sh bench:--workload,cfg4,--no-cpu-baseline,--no-secondary bench:--workload,cfg5,--no-cpu-baseline,--no-secondary multirank
for c in 8192 65536 262144; do timeout -s KILL 300 python tools/rank_probe.py $c 8 1 7; done > gpurun_out/rank_masked.log 2>&1
for c in 16384 65536; do timeout -s KILL 300 python tools/rank_probe.py $c 8 0 7; done > gpurun_out/rank_unmasked.log 2>&1
timeout -s KILL 600 python tools/masked_bwd_probe.py 524288 > gpurun_out/masked_bwd.log 2>&1
bash tools/gpu.sh tests smoke
ls -la gpurun_out/*.ncu-rep
