"""cfg3 (masked, T=1, N=512K) step: graph replay timed right after an idle
spin vs in steady state, and the per-kernel event sum in both conditions —
where the ~0.4 ms between the kernel sum and the back-to-back step goes."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, comm, lasp2  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

n, h, d = 524288, 16, 128
q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
ctx = comm.LocalRankContext()


def step():
    out, cache = lasp2.rank_forward(ctx, q, k, v, masked=True)
    g = lasp2.rank_backward(ctx, cache, do)
    return out, g


for _ in range(3):
    step()
torch.cuda.synchronize()
s2 = torch.cuda.Stream()
s2.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s2):
    step()
torch.cuda.current_stream().wait_stream(s2)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    step()
graph.replay()
torch.cuda.synchronize()


def timed(fn, k, sleep=False):
    if sleep:
        torch.cuda._sleep(int(6e8))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


def kernel_sum(k, sleep):
    _lib.PROFILER.reset(enabled=True)
    if sleep:
        torch.cuda._sleep(int(6e8))
    for _ in range(k):
        step()
    torch.cuda.synchronize()
    dur = _lib.PROFILER.durations_ms()
    _lib.PROFILER.reset(enabled=False)
    return sum(sum(x) for x in dur.values()) / k, {kk: round(sum(x) / k, 3) for kk, x in dur.items()}


for rep in range(2):
    print(f"graph after idle spin, 10 steps: {timed(graph.replay, 10, sleep=True):.3f} ms")
    print(f"graph steady, 20 steps:          {timed(graph.replay, 20):.3f} ms")
    print(f"graph steady, 60 steps:          {timed(graph.replay, 60):.3f} ms")
    print(f"eager steady, 20 steps:          {timed(step, 20):.3f} ms")
    ks, det = kernel_sum(10, True)
    print(f"kernel sum after idle spin:      {ks:.3f} ms {det}")
    ks, det = kernel_sum(20, False)
    print(f"kernel sum steady:               {ks:.3f} ms {det}")
