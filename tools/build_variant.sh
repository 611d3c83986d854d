#!/bin/bash
# Build the library with extra defines into ab_so/NAME.so (A/B variants for tools/gpu.sh ab:),
# then rebuild the default library in-tree.
#   bash tools/build_variant.sh NAME "DEFINE1 DEFINE2" [trace]
set -e
cd "$(dirname "$0")/.."
name=$1; defs=$2
if [ -n "$3" ]; then export LASP2_TRACE=1; fi
LASP2_DEFINES="$defs" python -m paper_2502_07563_b200.build > /dev/null
mkdir -p ab_so && cp paper_2502_07563_b200/liblasp2_b200.so "ab_so/$name.so"
unset LASP2_TRACE
python -m paper_2502_07563_b200.build > /dev/null
echo "ab_so/$name.so"
