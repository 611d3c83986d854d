"""Per-kernel device times (sleep-queued CUDA events) of one rank's fwd+bwd at chunk C in a
T-rank world, on one GPU: the state exchange is replaced by a local tensor of the right shape
(same kernels, no collective). Also the CUDA-graph step time.

usage: python tools/rank_probe.py C T masked(0/1) [rank] [LASP2_SWITCH=0|1 ...]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, comm  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402
from paper_2502_07563_b200.lasp2 import rank_backward, rank_forward  # noqa: E402

c = int(sys.argv[1]); world = int(sys.argv[2]); masked = sys.argv[3] == "1"
rank = int(sys.argv[4]) if len(sys.argv) > 4 else world - 1
for kv in sys.argv[5:]:  # module switches for A/B, e.g. FLAT_FOLD_IN_PHASE2=0
    key, val = kv.split("=")
    import paper_2502_07563_b200.lasp2 as _l2  # noqa: E402
    setattr(_l2, key, bool(int(val)))


class FakeWorld(comm.LocalRankContext):
    """sp_size T, position `rank`: all_gather returns this rank's payload in every slot."""
    sp_position = rank
    sp_size = world
    sp_peers = tuple(range(world))

    def all_gather_async(self, payload, tag=""):
        self._account("all_gather", payload)
        out = payload.unsqueeze(0).expand(world, *payload.shape).contiguous()

        class _D:
            def wait(s):
                return out
        return _D()


ctx = FakeWorld()
q, k, v, do = (gen_slots_device(0, 1, 16, c, 128, t, row_offset=rank * c) for t in ("q", "k", "v", "do"))


def step():
    out, cache = rank_forward(ctx, q, k, v, masked=masked)
    g = rank_backward(ctx, cache, do)
    return out, g.dq, g.dk, g.dv


for _ in range(5):
    step()
torch.cuda.synchronize()
_lib.PROFILER.reset(enabled=True)
torch.cuda._sleep(int(3e8))
reps = 20
for _ in range(reps):
    step()
torch.cuda.synchronize()
d = {kk: sum(x) / reps for kk, x in _lib.PROFILER.durations_ms().items()}
_lib.PROFILER.reset(enabled=False)
unit = 16 * c * 128 * 2 / 1e9
tot = sum(d.values())
print(f"C={c} T={world} rank={rank} masked={masked}: kernel sum {tot * 1e3:.1f} us "
      f"({11 * unit / tot * 1e3:.0f} GB/s of the 11-unit minimum)")
for kk, x in sorted(d.items(), key=lambda z: -z[1]):
    print(f"   {kk:40s} {x * 1e3:8.1f} us")
s2 = torch.cuda.Stream()
s2.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s2):
    step()
torch.cuda.current_stream().wait_stream(s2)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    g.replay()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 50
print(f"   graph step {ms * 1e3:.1f} us = {11 * unit / ms * 1e3:.0f} GB/s minimal bytes, {c / ms * 1e3 / 1e6:.1f} M tok/s/GPU")
