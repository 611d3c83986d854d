"""Per-launch time vs N for the streaming kernels: fixed cost + per-block cost fit."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(3e8))
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


h, d = 16, 128
rows = []
for n in (32768, 65536, 131072, 262144, 524288):
    q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
    nseg = ops.num_segments(k)
    m = torch.randn((1, h, d, d), device="cuda")
    unit = h * n * d * 2 / 1e9
    t_seg = timeit(lambda: ops.segment_states(k, v, nseg))
    t_app = timeit(lambda: ops.apply_state(q, m))
    t_sa = timeit(lambda: ops.state_apply(q, do, m, nseg))
    t_a2 = timeit(lambda: ops.apply_state2(v, k, m))
    rows.append((n, t_seg, t_app, t_sa, t_a2))
    print(f"N={n:7d} seg {t_seg*1e3:7.1f}us ({2*unit/t_seg*1e3:5.0f} GB/s)  apply {t_app*1e3:7.1f}us "
          f"({2*unit/t_app*1e3:5.0f})  state_apply {t_sa*1e3:7.1f}us ({3*unit/t_sa*1e3:5.0f})  "
          f"apply2 {t_a2*1e3:7.1f}us ({4*unit/t_a2*1e3:5.0f})")
(n0, *a), (n1, *b) = rows[1], rows[-1]
for name, x0, x1 in zip(("seg", "apply", "state_apply", "apply2"), a, b):
    per = (x1 - x0) / (n1 - n0)
    print(f"{name:12s} fixed {(x0 - per * n0) * 1e3:6.1f} us  per-128-token-block {per * 128 * 1e3:7.3f} us")
