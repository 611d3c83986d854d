#!/bin/bash
# A/B of two prebuilt libraries (ab_so/old.so, ab_so/new.so) on the same box, alternating
cd "${GRAFT_REPO_ROOT:-.}"
WL=${1:-cfg3}
for rep in 1 2; do
  for v in old new; do
    cp ab_so/$v.so paper_2502_07563_b200/liblasp2_b200.so
    timeout -s KILL 300 python bench.py --workload $WL --no-cpu-baseline --no-secondary 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$WL', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['per_kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
  done
done
