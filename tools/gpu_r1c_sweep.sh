#!/bin/bash
# cfg5 per-rank sweep + bench line with the longer e2e pipeline
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python tools/cfg5_sweep.py > gpurun_out/cfg5_sweep.log 2>&1
timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
cat gpurun_out/cfg5_sweep.log; python -c "
import json; d=json.loads(open('gpurun_out/bench_e2e.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['secondary']['e2e'])"
