#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
bash tools/gpu_ab_so.sh cfg3
for v in old new; do
  cp ab_so/$v.so paper_2502_07563_b200/liblasp2_b200.so
  echo "== $v"; timeout -s KILL 300 python tools/cfg5_sweep.py 65536 262144 2>&1 | grep -A1 "sequential t=7" | grep graph
done
LASP2_DEFINES=LASP2_SPAN python -m paper_2502_07563_b200.build > /dev/null 2>&1
timeout -s KILL 200 python tools/cta_phase_probe.py 8192 2>&1
