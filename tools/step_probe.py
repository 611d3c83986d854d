"""Step time of a bench workload three ways: eager launches, CUDA-graph replay,
and the sum of per-kernel CUDA-event durations (sleep-queued)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, comm  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402
from paper_2502_07563_b200.lasp2 import rank_backward, rank_forward  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
masked = (sys.argv[2] if len(sys.argv) > 2 else "1") == "1"
q, k, v, do = (gen_slots_device(0, 1, 16, n, 128, t) for t in ("q", "k", "v", "do"))
ctx = comm.LocalRankContext()


def step():
    out, cache = rank_forward(ctx, q, k, v, masked=masked)
    g = rank_backward(ctx, cache, do)
    return out, g.dq, g.dk, g.dv


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


eager = timed(step)
_lib.PROFILER.reset(enabled=True)
torch.cuda._sleep(int(3e8))
for _ in range(5):
    step()
torch.cuda.synchronize()
d = _lib.PROFILER.durations_ms()
_lib.PROFILER.reset(enabled=False)
ksum = sum(sum(x) for x in d.values()) / 5
s2 = torch.cuda.Stream()
s2.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s2):
    step()
torch.cuda.current_stream().wait_stream(s2)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
graph = timed(g.replay)
print(f"n={n} masked={masked}: eager {eager:.3f} ms  graph {graph:.3f} ms  kernel-sum {ksum:.3f} ms")
print({kk: round(sum(x) / 5, 4) for kk, x in d.items()})
