"""Phase timeline of the world-of-one persistent kernels (globaltimer per CTA)
and event timing against the per-step kernels at the cfg2 shape."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
h, d = 16, 128
q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
unit = q.numel() * 2


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for i in range(reps):
        ev[2 * i].record()
        fn()
        ev[2 * i + 1].record()
    torch.cuda.synchronize()
    ts = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps))
    return ts[len(ts) // 2]


out, m = ops.nomask_forward_local(q, k, v)
fwd = timeit(lambda: ops.nomask_forward_local(q, k, v))
bwd = timeit(lambda: ops.nomask_backward_local(q, k, v, do, m))
print(f"local fwd {fwd*1e3:.1f} us ({4*unit/fwd/1e6:.0f} GB/s)   local bwd {bwd*1e3:.1f} us ({7*unit/bwd/1e6:.0f} GB/s)")


def old_fwd():
    _, mt, _ = ops.chunk_states(k, v)
    return ops.apply_state(q, mt)


def old_bwd():
    nseg = ops.num_segments(q)
    gseg, dq = ops.state_apply(q, do, m, nseg)
    g = ops.scan_segments(gseg, reverse=False, data_dtype=q.dtype)
    return ops.apply_state2(v, k, g)


print(f"step fwd {timeit(old_fwd)*1e3:.1f} us   step bwd {timeit(old_bwd)*1e3:.1f} us")
print(f"segment_states {timeit(lambda: ops.segment_states(k, v, ops.num_segments(k)))*1e3:.1f} us  "
      f"apply_state {timeit(lambda: ops.apply_state(q, m))*1e3:.1f} us  "
      f"apply2 {timeit(lambda: ops.apply_state2(v, k, m))*1e3:.1f} us")

buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
names = ["start", "p1_done", "barrier1", "reduced", "img_ready", "p2_done", "end"]
for label, fn in (("fwd", lambda: ops.nomask_forward_local(q, k, v)),
                  ("bwd", lambda: ops.nomask_backward_local(q, k, v, do, m))):
    buf.zero_()
    torch.cuda.synchronize()
    _lib.call("lasp2_debug_trace", buf.data_ptr())
    fn()
    torch.cuda.synchronize()
    _lib.call("lasp2_debug_trace", None)
    t = buf.view(148, 8).cpu()
    t0 = t[:, 0][t[:, 0] > 0].min().item()
    print(f"--- {label} (us from first CTA start): min / median / max over CTAs")
    for i, nm in enumerate(names):
        col = t[:, i]
        col = col[col > 0].double() - t0
        if col.numel():
            print(f"   {nm:10s} {col.min().item()/1e3:8.1f} {col.median().item()/1e3:8.1f} {col.max().item()/1e3:8.1f}")
    nb = (n + 127) // 128
    F = nb * h
    p2 = (t[:, 5] - t[:, 4]).double() / 1e3
    p1 = (t[:, 1] - t[:, 0]).double() / 1e3
    order = torch.argsort(p2, descending=True)
    print("   slowest phase-2 CTAs (cta, f0 % nb, blocks, p1 us, p2 us):",
          [(int(c), (int(c) * F // 148) % nb, ((int(c) + 1) * F // 148) - (int(c) * F // 148), round(p1[c].item(), 1),
            round(p2[c].item(), 1)) for c in order[:12]])
    print("   fastest:", [(int(c), round(p2[c].item(), 1)) for c in order[-5:]])
