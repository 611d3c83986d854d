#!/bin/bash
# ncu --set full of one rank's kernels at the per-rank chunk of every N > 1 bench run (so bench.py can
# report roofline.traffic for N = 2 / 4 / 8): cfg2 unmasked phase kernels, cfg3 masked passes
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
run() {  # name regex count C T masked
  timeout -s KILL 900 ncu --set full --clock-control none -k "regex:$2" -c "$3" -o "gpurun_out/$1" -f \
    python tools/rank_probe.py "$4" "$5" "$6" 1 > "gpurun_out/$1.log" 2>&1
  echo "$1 rc=$?"
}
run ncu_cfg2_c65536 tc_flat_kernel 4 65536 2 0
run ncu_cfg2_c32768 tc_flat_kernel 4 32768 4 0
run ncu_cfg3_c262144 "causal_chunk|segment_states" 4 262144 2 1
run ncu_cfg3_c131072 "causal_chunk|segment_states" 4 131072 4 1
run ncu_cfg3_c65536 "causal_chunk|segment_states" 4 65536 8 1
ls -la gpurun_out/*.ncu-rep
