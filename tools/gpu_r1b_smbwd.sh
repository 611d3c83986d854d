#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"tc_softmax_bwd" -c 1 \
   -o gpurun_out/r1b_softmax_bwd -f python tools/perf_probe.py 0 softmax 32768 > gpurun_out/ncu_softmax_bwd.log 2>&1
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_clk.json 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_clk.json").read().strip().splitlines()[-1])
print("cfg2", d["ms_per_step"], d["clocks"])
print("cfg3", d["secondary"]["ms_per_step"], d["secondary"]["clocks"])
PY
