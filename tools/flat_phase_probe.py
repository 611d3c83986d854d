"""Per-CTA globaltimer timeline of the T > 1 unmasked phase kernels (lasp2_nomask_*_phase)
at one rank's chunk C: where a phase launch spends its time at small C.

usage: python tools/flat_phase_probe.py [C]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
h, d = 16, 128
q, k, v, do = (gen_slots_device(0, 1, h, c, d, t) for t in ("q", "k", "v", "do"))
m = torch.empty((1, h, d, d), dtype=torch.float32, device="cuda")
ops.nomask_forward_phase(q, k, v, m, 1)
mf = m.clone()
names = ["start", "p1_done", "barrier1", "reduced", "img_ready", "p2_done", "end"]
runs = {"fwd phase1": lambda: ops.nomask_forward_phase(q, k, v, m, 1),
        "fwd phase2": lambda: ops.nomask_forward_phase(q, k, v, mf, 2),
        "bwd phase1": lambda: ops.nomask_backward_phase1(q, do, mf),
        "bwd phase2": lambda: ops.nomask_backward_phase2(v, k, mf)}
buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
for label, fn in runs.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    ev = a.elapsed_time(b) / 20 * 1e3
    buf.zero_()
    torch.cuda.synchronize()
    _lib.call("lasp2_debug_trace", buf.data_ptr())
    fn()
    torch.cuda.synchronize()
    _lib.call("lasp2_debug_trace", None)
    t = buf.view(148, 8).cpu()
    t0 = t[:, 0][t[:, 0] > 0].min().item()
    print(f"--- {label}: {ev:.1f} us per launch back to back; stamps (us from first CTA start) min / median / max")
    for i, nm in enumerate(names):
        col = t[:, i]
        col = col[col > 0].double() - t0
        if col.numel():
            print(f"   {nm:10s} {col.min().item()/1e3:8.1f} {col.median().item()/1e3:8.1f} {col.max().item()/1e3:8.1f}")
