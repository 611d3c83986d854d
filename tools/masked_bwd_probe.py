"""Masked backward variants at one rank's shape: per-kernel CUDA-event times (sleep-queued) of
the default (dq_chunk + dkdv pair) and the single-launch forward-walking triple
(lasp2_backward_chunk_fwd, kMode 4; lasp2.MASKED_BWD_FUSED).

usage: python tools/masked_bwd_probe.py [N] [T]   (rank t = T-1 of a T-rank world: both folds)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, lasp2  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402
from paper_2502_07563_b200.lasp2 import rank_backward, rank_forward  # noqa: E402
from paper_2502_07563_b200 import comm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
q, k, v, do = (gen_slots_device(0, 1, 16, n, 128, t) for t in ("q", "k", "v", "do"))
ctx = comm.LocalRankContext()
unit = 16 * n * 128 * 2 / 1e9
for fused in (False, True, False, True):
    lasp2.MASKED_BWD_FUSED = fused
    out, cache = rank_forward(ctx, q, k, v, masked=True)
    for _ in range(3):
        rank_backward(ctx, cache, do)
    torch.cuda.synchronize()
    _lib.PROFILER.reset(enabled=True)
    torch.cuda._sleep(int(3e8))
    for _ in range(5):
        rank_backward(ctx, cache, do)
    torch.cuda.synchronize()
    d = {kk: sum(x) / 5 for kk, x in _lib.PROFILER.durations_ms().items()}
    _lib.PROFILER.reset(enabled=False)
    tot = sum(d.values())
    print(f"fused={fused} backward kernel sum {tot:.3f} ms ({11 if not fused else 9} units: "
          f"{(11 if not fused else 9) * unit / tot * 1e3:.0f} GB/s) " +
          " ".join(f"{kk}={x:.3f}" for kk, x in d.items()))
