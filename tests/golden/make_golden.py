"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports laspsim from /root/reference/pkg/src (read-only), runs the
reference's own world drivers on small cases from its test grids
(pkg/tests/test_lasp2.py, test_acceptance.py, test_standard_sp.py) and on a
row-subsampled cfg1 case, and writes tests/golden/reference_cases.npz.
The fixtures travel with the repo; nothing at test time reads /root/reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "reference_cases.npz"

LASP_CASES = [  # (n, d, t, batch, heads, seed)
    (8, 4, 1, 1, 1, 0), (8, 4, 2, 1, 1, 0), (16, 8, 4, 1, 1, 0), (16, 4, 8, 1, 1, 0),
    (64, 16, 4, 1, 1, 0), (256, 16, 8, 1, 1, 0), (256, 4, 2, 1, 1, 0), (8, 4, 4, 2, 3, 5),
    (256, 32, 4, 1, 2, 7),
]
CP_CASES = [(8, 4, 2, 1, 1, 0), (16, 8, 4, 1, 1, 0), (16, 4, 2, 1, 1, 0), (8, 4, 4, 2, 2, 3), (256, 32, 4, 1, 2, 1)]
CFG1 = (4096, 64, 2, 1, 4, 0)  # B=1 H=4 d=64 N=4096 W=2
CFG1_ROWS = np.arange(0, 4096, 127)


def main() -> None:
    sys.path.insert(0, str(REF))
    from laspsim.datagen import gen_slots, qkv_slots
    from laspsim.lasp2 import ChunkedSequence, lasp2_iteration
    from laspsim.standard_sp import cp_iteration

    def inputs(n, d, b, h, seed):
        q, k, v = qkv_slots(seed, b, h, n, d)
        return q, k, v, gen_slots(seed, b, h, n, d, "do")

    cat = lambda xs: np.concatenate(xs, axis=2)  # noqa: E731
    data = {}
    for masked in (True, False):
        for (n, d, t, b, h, seed) in LASP_CASES:
            q, k, v, do = inputs(n, d, b, h, seed)
            it = lasp2_iteration(ChunkedSequence(q, k, v, t), do, masked)
            key = f"lasp2_{'m' if masked else 'u'}_{n}_{d}_{t}_{b}_{h}_{seed}"
            data[key + "_out"] = cat(it.outputs)
            data[key + "_dq"] = cat([g.dq for g in it.grads])
            data[key + "_dk"] = cat([g.dk for g in it.grads])
            data[key + "_dv"] = cat([g.dv for g in it.grads])
            data[key + "_launches"] = np.array([it.run.stats.allgather_launches, it.run.stats.bytes_sent])
    for causal in (True, False):
        for (n, d, t, b, h, seed) in CP_CASES:
            q, k, v, do = inputs(n, d, b, h, seed)
            it = cp_iteration(ChunkedSequence(q, k, v, t), do, causal)
            key = f"cp_{'c' if causal else 'n'}_{n}_{d}_{t}_{b}_{h}_{seed}"
            data[key + "_out"] = cat(it.outputs)
            data[key + "_dq"] = cat([g.dq for g in it.grads])
            data[key + "_dk"] = cat([g.dk for g in it.grads])
            data[key + "_dv"] = cat([g.dv for g in it.grads])
    n, d, t, b, h, seed = CFG1
    q, k, v, do = inputs(n, d, b, h, seed)
    it = lasp2_iteration(ChunkedSequence(q, k, v, t), do, True)
    for name, arr in (("out", cat(it.outputs)), ("dq", cat([g.dq for g in it.grads])),
                      ("dk", cat([g.dk for g in it.grads])), ("dv", cat([g.dv for g in it.grads]))):
        data[f"cfg1_{name}_rows"] = arr[:, :, CFG1_ROWS, :]
        data[f"cfg1_{name}_sum"] = np.array([arr.sum(), (arr * arr).sum(), np.abs(arr).max()])
    data["cfg1_rows"] = CFG1_ROWS
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(data)} arrays)")
    hybrid_cases()
    lasp1_cases()


# (pattern, n, d, chunks, batch, heads, seed, causal): test_hybrid.py grids plus two larger stacks
HYBRID_CASES = [(p, 16, 4, t, 1, 1, 2, True) for p in ("L", "N", "LN", "LLLN", "LNLN LNLN") for t in (1, 2, 4)] + [
    ("LN", 8, 4, 2, 1, 1, 5, False), ("LN", 8, 4, 2, 2, 2, 6, True),
    ("LLN", 256, 32, 2, 1, 2, 11, True), ("LN", 256, 32, 4, 1, 2, 12, False),
]


def hybrid_key(pattern, n, d, t, b, h, seed, causal):
    return f"hy_{pattern.replace(' ', '_')}_{n}_{d}_{t}_{b}_{h}_{seed}_{'c' if causal else 'n'}"


def hybrid_cases() -> None:
    """Reference hybrid_iteration outputs (hybrid.py:284-303) -> tests/golden/hybrid_cases.npz."""
    from laspsim.datagen import gen_slots
    from laspsim.hybrid import ModelSpec, hybrid_iteration

    out_path = OUT.parent / "hybrid_cases.npz"
    data = {}
    for case in HYBRID_CASES:
        pattern, n, d, t, b, h, seed, causal = case
        spec = ModelSpec(pattern, dim=d, heads=h, batch=b, seed=seed)
        x = gen_slots(seed, b, h, n, d, "x")
        dy = gen_slots(seed, b, h, n, d, "dy")
        it = hybrid_iteration(spec, x, dy, t, causal=causal)
        key = hybrid_key(*case)
        data[key + "_out"] = np.concatenate(it.outputs, axis=2)
        data[key + "_dx"] = np.concatenate(it.d_x, axis=2)
        data[key + "_dw"] = np.stack([np.stack(w) for w in it.d_weights])
        data[key + "_ledger"] = np.array([it.run.stats.allgather_launches, it.run.stats.p2p_sends])
    np.savez_compressed(out_path, **data)
    print(f"wrote {out_path} ({out_path.stat().st_size} bytes, {len(data)} arrays)")


# (n, d, t, batch, heads, seed): test_lasp1.py grids plus a multi-slot and a larger case
LASP1_CASES = [(8, 4, 2, 1, 1, 0), (8, 8, 4, 1, 1, 0), (16, 4, 4, 1, 1, 0), (16, 8, 8, 1, 1, 0),
               (16, 4, 4, 2, 3, 2), (256, 32, 4, 1, 2, 9)]


def lasp1_cases() -> None:
    """Reference lasp1_iteration outputs (lasp1.py:191-210) -> tests/golden/lasp1_cases.npz."""
    from laspsim.datagen import gen_slots, qkv_slots
    from laspsim.lasp1 import lasp1_iteration
    from laspsim.lasp2 import ChunkedSequence

    out_path = OUT.parent / "lasp1_cases.npz"
    data = {}
    cat = lambda xs: np.concatenate(xs, axis=2)  # noqa: E731
    for masked in (True, False):
        for (n, d, t, b, h, seed) in LASP1_CASES:
            q, k, v = qkv_slots(seed, b, h, n, d)
            do = gen_slots(seed, b, h, n, d, "do")
            it = lasp1_iteration(ChunkedSequence(q, k, v, t), do, masked)
            key = f"l1_{'m' if masked else 'u'}_{n}_{d}_{t}_{b}_{h}_{seed}"
            data[key + "_out"] = cat(it.outputs)
            for nm in ("dq", "dk", "dv"):
                data[f"{key}_{nm}"] = cat([getattr(g, nm) for g in it.grads])
            data[key + "_through"] = it.caches[-1].state_through
            st = it.run.stats
            data[key + "_ledger"] = np.array([st.p2p_sends, st.allgather_launches, st.communication_steps,
                                              st.bytes_sent])
    np.savez_compressed(out_path, **data)
    print(f"wrote {out_path} ({out_path.stat().st_size} bytes, {len(data)} arrays)")


# Simulated-clock cases: (method, n, d, t, world, batch, heads, masked/causal, pattern,
# latency_per_launch, latency_per_byte). The reference clock depends only on the
# schedule and the payload sizes, so these pin comm.py:7-12's model for every driver.
CLOCK_CASES = [
    ("lasp2", 16, 4, 4, 4, 1, 1, True, "", 10.0, 1 / 1024), ("lasp2", 16, 4, 4, 4, 1, 1, False, "", 10.0, 1 / 1024),
    ("lasp2", 32, 8, 8, 8, 2, 3, True, "", 10.0, 1 / 1024), ("lasp2", 32, 4, 4, 8, 1, 1, True, "", 3.0, 0.25),
    ("lasp2", 32, 4, 8, 8, 1, 1, True, "", 10.0, 0.0), ("lasp2_overlap", 16, 4, 4, 4, 1, 1, True, "", 10.0, 1 / 1024),
    ("lasp1", 16, 4, 4, 4, 1, 1, True, "", 10.0, 1 / 1024), ("lasp1", 16, 4, 4, 4, 1, 1, False, "", 10.0, 1 / 1024),
    ("lasp1", 32, 8, 8, 8, 2, 3, True, "", 10.0, 1 / 1024), ("lasp1", 32, 4, 8, 8, 1, 1, True, "", 10.0, 0.0),
    ("lasp1", 32, 4, 4, 8, 1, 1, True, "", 3.0, 0.25),
    ("cp", 16, 4, 4, 4, 1, 1, True, "", 10.0, 1 / 1024), ("cp", 16, 4, 2, 4, 2, 2, False, "", 10.0, 1 / 1024),
    ("hybrid", 16, 4, 4, 4, 1, 1, True, "LLLN", 10.0, 1 / 1024), ("hybrid", 16, 8, 2, 2, 1, 2, True, "LN LN", 2.0, 0.5),
]


def clock_cases() -> None:
    """Reference WorldRun.simulated_time for every driver -> tests/golden/clock_cases.json."""
    import json

    from laspsim import comm
    from laspsim.datagen import gen_slots, qkv_slots
    from laspsim.hybrid import ModelSpec, hybrid_iteration
    from laspsim.lasp1 import lasp1_iteration
    from laspsim.lasp2 import ChunkedSequence, lasp2_iteration
    from laspsim.standard_sp import cp_iteration

    rows = []
    for case in CLOCK_CASES:
        method, n, d, t, world, b, h, masked, pattern, lat_l, lat_b = case
        cfg = comm.WorldConfig(world_size=world, sp_size=t, element_bytes=8,
                               latency_per_launch=lat_l, latency_per_byte=lat_b)
        if method == "hybrid":
            spec = ModelSpec(pattern, dim=d, heads=h, batch=b, seed=0)
            x, dy = gen_slots(0, b, h, n, d, "x"), gen_slots(0, b, h, n, d, "dy")
            run = hybrid_iteration(spec, x, dy, t, masked, cfg).run
        else:
            q, k, v = qkv_slots(0, b, h, n, d)
            do = gen_slots(0, b, h, n, d, "do")
            seq = ChunkedSequence(q, k, v, t)
            if method == "lasp2_overlap":
                run = lasp2_iteration(seq, do, masked, cfg, overlap=True).run
            else:
                driver = {"lasp2": lasp2_iteration, "lasp1": lasp1_iteration, "cp": cp_iteration}[method]
                run = driver(seq, do, masked, cfg).run
        rows.append({"case": list(case), "simulated_time": run.simulated_time,
                     "communication_steps": run.stats.communication_steps, "bytes_sent": run.stats.bytes_sent})
    out_path = OUT.parent / "clock_cases.json"
    out_path.write_text("[\n" + ",\n".join(json.dumps(r) for r in rows) + "\n]\n")
    print(f"wrote {out_path} ({len(rows)} cases)")


def costmodel_table() -> None:
    """The reference CLI's default cost table (cli.py:765-810) -> tests/golden/costmodel_default.csv."""
    from laspsim.cli import main as cli_main

    out_path = OUT.parent / "costmodel_default.csv"
    assert cli_main(["costmodel", "--out", str(out_path)]) == 0
    print(f"wrote {out_path}")


if __name__ == "__main__":
    if sys.argv[1:] == ["costmodel"]:
        sys.path.insert(0, str(REF))
        costmodel_table()
    elif sys.argv[1:] == ["clock"]:
        sys.path.insert(0, str(REF))
        clock_cases()
    elif sys.argv[1:] == ["hybrid"]:
        sys.path.insert(0, str(REF))
        hybrid_cases()
    elif sys.argv[1:] == ["lasp1"]:
        sys.path.insert(0, str(REF))
        lasp1_cases()
    else:
        main()
