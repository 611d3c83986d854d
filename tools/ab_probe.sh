#!/bin/bash
# Run one command against several prebuilt libraries (ab_so/NAME.so), twice, interleaved:
#   bash tools/ab_probe.sh "old new" python tools/masked_bwd_probe.py 524288
# Output lines are prefixed with the variant name; the in-tree library is restored at the end.
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
vars=$1; shift
cp paper_2502_07563_b200/liblasp2_b200.so /tmp/lasp2_default.so
for rep in 1 2; do
  for v in $vars; do
    cp "ab_so/$v.so" paper_2502_07563_b200/liblasp2_b200.so
    timeout -s KILL 300 "$@" 2>&1 | sed "s/^/$v /"
  done
done
cp /tmp/lasp2_default.so paper_2502_07563_b200/liblasp2_b200.so
