"""Host-side cost per call (no device sync inside the loop) of the layer entry points."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import comm, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402
from paper_2502_07563_b200.lasp2 import rank_backward, rank_forward  # noqa: E402

n = 8192
q, k, v, do = (gen_slots_device(0, 1, 16, n, 128, t) for t in ("q", "k", "v", "do"))
ctx = comm.LocalRankContext()
out, m = ops.nomask_forward_local(q, k, v)
nseg = ops.num_segments(q)
seg = ops.segment_states(k, v, nseg)


def host(label, fn, reps=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label:28s} host {1e6 * (t1 - t0) / reps:8.1f} us/call   (+drain {1e3 * (t2 - t1):.2f} ms)")


host("torch.empty_like", lambda: torch.empty_like(q))
host("nomask_forward_local", lambda: ops.nomask_forward_local(q, k, v))
host("nomask_backward_local", lambda: ops.nomask_backward_local(q, k, v, do, m))
host("segment_states", lambda: ops.segment_states(k, v, nseg))
host("causal_chunk", lambda: ops.causal_chunk(q, k, v, seg, None, nseg))
host("apply_state", lambda: ops.apply_state(q, m))
host("fold(prefix)", lambda: ops.prefix_states(m.unsqueeze(0), 1))
host("rank fwd+bwd unmasked", lambda: rank_backward(ctx, rank_forward(ctx, q, k, v, masked=False)[1], do))
host("rank fwd+bwd masked", lambda: rank_backward(ctx, rank_forward(ctx, q, k, v, masked=True)[1], do))
