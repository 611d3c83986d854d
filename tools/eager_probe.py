"""Where does eager time go at the cfg2 size? host vs device per call."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import comm, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

n = 131072
q, k, v, do = (gen_slots_device(0, 1, 16, n, 128, t) for t in ("q", "k", "v", "do"))
out, m = ops.nomask_forward_local(q, k, v)
pre = [torch.empty_like(q) for _ in range(4)]


def run(label, fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    hs = []
    ev[0].record()
    for i in range(reps):
        h = time.perf_counter()
        fn()
        hs.append(time.perf_counter() - h)
        ev[i + 1].record()
    torch.cuda.synchronize()
    gaps = [ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]
    print(f"{label:34s} device/call {sum(gaps)/reps:.3f} ms  host/call {1e3*sum(hs)/reps:.3f} ms  "
          f"per-call device {[round(g, 3) for g in gaps[:5]]}")


from paper_2502_07563_b200.lasp2 import rank_backward, rank_forward  # noqa: E402
ctx = comm.LocalRankContext()
_, cache = rank_forward(ctx, q, k, v, masked=False)
run("rank_forward unmasked", lambda: rank_forward(ctx, q, k, v, masked=False))
run("rank_backward unmasked", lambda: rank_backward(ctx, cache, do))
run("rank step unmasked", lambda: rank_backward(ctx, rank_forward(ctx, q, k, v, masked=False)[1], do))
run("forward_local", lambda: ops.nomask_forward_local(q, k, v))
run("backward_local", lambda: ops.nomask_backward_local(q, k, v, do, m))
run("fwd+bwd local", lambda: ops.nomask_backward_local(q, k, v, do, ops.nomask_forward_local(q, k, v)[1]))
run("apply_state", lambda: ops.apply_state(q, m))
run("apply_state into preallocated", lambda: ops.apply_state(q, m, out=pre[0]))
run("segment_states", lambda: ops.segment_states(k, v, 9))
run("torch add (512MB)", lambda: torch.add(q, k, out=pre[1]))
