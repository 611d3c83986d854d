"""Per-CTA start / end (globaltimer) of the masked causal-family kernels at the
cfg3 shape: how much of each kernel is the tail of the slowest CTAs."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
h, d = 16, 128
q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
nseg = ops.num_segments(k)
seg = ops.segment_states(k, v, nseg)
ops.scan_segments(seg, False, k.dtype)
dq, gseg = ops.dq_chunk(q, k, v, do, seg, None, nseg)
ops.scan_segments(gseg, True, q.dtype)
buf = torch.zeros(2 * 2 * nseg * h + 64, dtype=torch.int64, device="cuda")
runs = {"causal_chunk (fwd)": lambda: ops.causal_chunk(q, k, v, seg, None, nseg),
        "dq_chunk": lambda: ops.dq_chunk(q, k, v, do, seg, None, nseg),
        "dkdv_chunk": lambda: ops.dkdv_chunk(q, k, v, do, gseg, None, nseg)}
for name, fn in runs.items():
    for rep in range(3):
        fn()
        torch.cuda.synchronize()
        buf.zero_()
        _lib.call("lasp2_debug_trace", buf.data_ptr())
        fn()
        torch.cuda.synchronize()
        _lib.call("lasp2_debug_trace", None)
        t = buf.view(-1, 2).cpu()
        t = t[t[:, 0] > 0]
        t0 = int(t[:, 0].min())
        start, end = (t[:, 0] - t0).double() / 1e3, (t[:, 1] - t0).double() / 1e3
        dur = end - start
        s_end = end.sort().values
        print(f"{name:20s} ctas={len(t)} kernel={float(end.max()):.1f}us  end p0/p50/p90/p100 = "
              f"{float(s_end[0]):.1f}/{float(s_end[len(s_end)//2]):.1f}/{float(s_end[int(len(s_end)*0.9)]):.1f}/"
              f"{float(s_end[-1]):.1f}  start max {float(start.max()):.1f}  dur min/max {float(dur.min()):.1f}/"
              f"{float(dur.max()):.1f}  mean-end/max-end {float(end.mean()/end.max()):.3f}")
