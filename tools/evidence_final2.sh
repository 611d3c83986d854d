#!/bin/bash
# final check after the pair's multicast-only prefetch: bench line + launch list, ncu of the masked kernels,
# masked backward probe, cfg5 2M line, GPU suite + smoke
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
bash tools/gpu.sh bench launches
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"causal_chunk" -c 3 \
  -o gpurun_out/fin2_cfg3 -f python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_cfg3.log 2>&1
timeout -s KILL 600 python tools/masked_bwd_probe.py 524288 > gpurun_out/masked_bwd.log 2>&1
bash tools/gpu.sh bench:--workload,cfg5,--no-cpu-baseline,--no-secondary tests smoke
