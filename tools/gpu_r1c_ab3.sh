#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for v in old new old new; do
  cp ab_so/$v.so paper_2502_07563_b200/liblasp2_b200.so
  echo "== $v"; timeout -s KILL 300 python tools/cfg5_sweep.py 65536 2>&1 | grep -A1 "sequential t=7" | grep graph
  timeout -s KILL 300 python tools/cfg5_sweep.py --unmasked 131072 2>&1 | grep -A1 "t=7" | grep graph
done
cp ab_so/new.so paper_2502_07563_b200/liblasp2_b200.so
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lasp2.py -q -x -p no:cacheprovider 2>&1 | tail -2
