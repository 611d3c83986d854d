#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
for ns in "" 4 2 6; do
  echo "== NSEG=${ns:-default}"
  NSEG=$ns timeout -s KILL 300 python tools/cfg5_sweep.py 65536 131072 262144 524288 1048576 2>&1 | grep -A1 "sequential t=7" | grep graph
done
