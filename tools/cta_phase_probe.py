"""Where a masked causal-family CTA spends its time (diagnostic build
LASP2_DEFINES=LASP2_SPAN): globaltimer stamps per CTA at start, after the
prologue (barriers, TMEM alloc), after the epilogue's seed state, at the first
block's P, at the first block's O store, at the end of the block loop, after
the store drain, and at exit. Prints the median over CTAs of each interval (us).

    LASP2_DEFINES=LASP2_SPAN python -m paper_2502_07563_b200.build && python tools/cta_phase_probe.py 8192
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
h, d = 16, 128
q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
nseg = ops.num_segments(k)
seg = ops.segment_states(k, v, nseg)
ops.scan_segments(seg, False, k.dtype)
dq, gseg = ops.dq_chunk(q, k, v, do, seg, None, nseg)
ops.scan_segments(gseg, True, q.dtype)
buf = torch.zeros(16 * 2 * nseg * h + 64, dtype=torch.int64, device="cuda")
NAMES = ["prologue", "seed", "first P", "first O store", "rest of blocks", "store drain", "exit"]
runs = {"causal_chunk": lambda: ops.causal_chunk(q, k, v, seg, None, nseg),
        "dq_chunk": lambda: ops.dq_chunk(q, k, v, do, seg, None, nseg),
        "dkdv_chunk": lambda: ops.dkdv_chunk(q, k, v, do, gseg, None, nseg)}
for name, fn in runs.items():
    fn()
    torch.cuda.synchronize()
    buf.zero_()
    _lib.call("lasp2_debug_trace", buf.data_ptr())
    fn()
    torch.cuda.synchronize()
    _lib.call("lasp2_debug_trace", None)
    t = buf.view(-1, 16).cpu().double()
    t = t[t[:, 0] > 0]
    dt = (t[:, 1:8] - t[:, 0:7]) / 1e3
    med = dt.median(dim=0).values.tolist()
    tot = ((t[:, 7] - t[:, 0]) / 1e3).median().item()
    print(f"n={n} {name:13s} ctas={len(t)} median CTA {tot:.1f} us: " +
          "  ".join(f"{nm} {x:.1f}" for nm, x in zip(NAMES, med)))
    # inside the seed: epilogue start, chunk 0 loaded / stored, chunk 1 loaded / stored (from span 1)
    sub = [((t[:, i] - t[:, 1]) / 1e3).median().item() for i in (12, 8, 9, 10, 11, 2)]
    print("      seed detail (us after prologue): epi start %.1f  c0 loaded %.1f  c0 stored %.1f  "
          "c1 loaded %.1f  c1 stored %.1f  seed done %.1f" % tuple(sub))
