#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
run() { timeout -s KILL 300 env $1 python bench.py --workload cfg3 --no-cpu-baseline --no-secondary $2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],4), 'ksum', round(d['kernel_sum_ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['sm_min_mhz'])"; }
for rep in 1 2; do
  run "X=1" ""
  run "LASP2_NO_PDL=1" ""
  run "X=1" "--eager"
done
