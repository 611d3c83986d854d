"""Summarise ncu --set full captures (.ncu-rep) into profiles/ (text + json).

usage: python tools/ncu_summary.py OUT_PREFIX WORKLOAD rep1.ncu-rep [rep2 ...]
Writes OUT_PREFIX.txt (key metrics + top stall reasons per kernel) and merges
per-launch DRAM traffic into profiles/ncu_traffic.json keyed by C-ABI entry.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
]
ENTRY = {"tc_causal_chunk_kernel<0>": "lasp2_causal_chunk", "tc_causal_chunk_kernel<1>": "lasp2_dkdv_chunk",
         "tc_causal_chunk_kernel<2>": "lasp2_backward_chunk",
         "tc_causal_chunk_kernel<3>": "lasp2_dq_chunk", "tc_fused_apply_kernel<0>": "lasp2_state_apply",
         "tc_fused_apply_kernel<1>": "lasp2_apply_state2", "tc_apply_state": "lasp2_apply_state",
         "tc_segment_states": "lasp2_segment_states", "tc_softmax_fwd": "lasp2h_softmax_forward",
         "tc_softmax_bwd": "lasp2h_softmax_backward", "tc_flat_kernel<0>": "lasp2_nomask_forward_local",
         "tc_flat_kernel<1>": "lasp2_nomask_backward_local"}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def main():
    prefix = Path(sys.argv[1])
    lines = []
    traffic_path = Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    workload = sys.argv[2]
    traffic.setdefault(workload, {})
    # per-rank captures of T > 1 (workload "cfgN@C=..."): the flat kernels run as two phase
    # launches each, labelled in launch order like bench.py's profiler
    phased = "@C=" in workload
    seen: dict[str, int] = {}
    for rep in sys.argv[3:]:
        launches, units = raw(rep)
        for rec in launches:
            name = rec.get("Kernel Name", "?")
            phase_entry = None
            if phased and "tc_flat_kernel<" in name:
                kind = "forward" if "tc_flat_kernel<0>" in name else "backward"
                seen[kind] = seen.get(kind, 0) + 1
                phase_entry = f"lasp2_nomask_{kind}_phase{2 - seen[kind] % 2}"
            lines.append(f"== {Path(rep).name}: {name[:100]}")
            for k in KEYS:
                if k in rec:
                    lines.append(f"  {k:90s} {rec[k]:>16s} {units.get(k, '')}")
            pre = "smsp__average_warps_issue_stalled_"
            stalls = sorted(((float(v), k) for k, v in rec.items()
                             if k.startswith(pre) and k.endswith("_per_issue_active.ratio")
                             and v.replace('.', '', 1).isdigit()), reverse=True)[:8]
            if stalls:
                lines.append("  top stall reasons (warp cycles per issued instruction):")
                for v, k in stalls:
                    lines.append(f"    {k.replace(pre, '').replace('_per_issue_active.ratio', ''):40s} {v:8.2f}")
            try:
                rd = float(rec["dram__bytes_read.sum"]) * (1e9 if units["dram__bytes_read.sum"] == "Gbyte" else 1e6 if units["dram__bytes_read.sum"] == "Mbyte" else 1)
                wr = float(rec["dram__bytes_write.sum"]) * (1e9 if units["dram__bytes_write.sum"] == "Gbyte" else 1e6 if units["dram__bytes_write.sum"] == "Mbyte" else 1)
                if phase_entry is not None:
                    traffic[workload][phase_entry] = {"bytes_per_launch": rd + wr, "read": rd, "write": wr,
                                                      "source": str(prefix.name), "kernel": name[:80]}
                for key, entry in (() if phase_entry is not None else ENTRY.items()):
                    if key in name:
                        traffic[workload][entry] = {"bytes_per_launch": rd + wr, "read": rd, "write": wr,
                                          "source": str(prefix.name), "kernel": name[:80]}
            except (KeyError, ValueError):
                pass
    prefix.with_suffix(".txt").write_text("\n".join(lines) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
