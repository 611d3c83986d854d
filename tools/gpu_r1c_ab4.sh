#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for v in old new old new; do
  cp ab_so/$v.so paper_2502_07563_b200/liblasp2_b200.so
  echo "== $v"; timeout -s KILL 300 python tools/cfg5_sweep.py 65536 524288 2>&1 | grep -A1 "sequential t=7" | grep graph
done
bash tools/gpu_ab_so.sh cfg3
cp ab_so/new.so paper_2502_07563_b200/liblasp2_b200.so
timeout -s KILL 900 python -m pytest tests/test_gpu_lasp2.py tests/test_gpu_kernels.py tests/test_gpu_peer_exchange.py tests/test_gpu_acceptance.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -2
LASP2_DEFINES=LASP2_SPAN python -m paper_2502_07563_b200.build > /dev/null 2>&1
timeout -s KILL 200 python tools/cta_phase_probe.py 8192 2>&1
