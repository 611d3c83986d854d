"""One bench.py run of a workload, reduced to a line: step ms, per-kernel ms, SM clock (A/B helper).

usage: python tools/ab_bench.py WORKLOAD [extra bench args]"""
import json
import subprocess
import sys

wl = sys.argv[1]
r = subprocess.run([sys.executable, "bench.py", "--workload", wl, "--no-cpu-baseline", "--no-secondary", *sys.argv[2:]],
                   capture_output=True, text=True)
try:
    d = json.loads(r.stdout.strip().splitlines()[-1])
except Exception:
    print("failed", r.stderr[-600:])
    sys.exit(1)
print(wl, round(d["ms_per_step"], 4), {k: round(x, 4) for k, x in d["per_kernel_ms_per_step"].items()},
      d["clocks"]["sm_mhz"], d["clocks"].get("reasons"))
