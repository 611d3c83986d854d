"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of a
bench run: per kernel launch count, mean duration and share of the layer's
device time (datagen, sleeps and torch helpers excluded).

usage: python tools/launch_summary.py launches.csv "command line" > profiles/rNN_launch_list.txt
"""
import csv
import re
import sys
from collections import defaultdict

EXCLUDE = ("gen_slots", "sleep", "spin_kernel", "at::", "elementwise", "vectorized", "fill", "copy")


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value")}
    dur = defaultdict(list)
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]]
        if any(x in name for x in EXCLUDE):
            continue
        name = re.sub(r"\(.*", "", name).replace("lasp::", "")
        dur[name].append(float(r[ix["Metric Value"]]) / 1e3)
    total = sum(sum(v) for v in dur.values())
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none {cmd}")
    print("(cold-cache, serialised launches; shares over the layer's own kernels, datagen/sleep excluded)")
    for name, v in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
        print(f"{name:60s} n={len(v):4d} mean={sum(v)/len(v):10.1f} us  share={100*sum(v)/total:5.1f}%")


if __name__ == "__main__":
    main()
