"""The per-rank layer step captured as a CUDA graph replays to the eager result."""
import pytest
import torch

from paper_2502_07563_b200 import comm
from paper_2502_07563_b200.datagen import gen_slots_device
from paper_2502_07563_b200.lasp2 import rank_backward, rank_forward

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("masked", [True, False])
def test_graph_replay_matches_eager(masked):
    ctx = comm.LocalRankContext()
    q, k, v, do = (gen_slots_device(0, 1, 4, 8192, 128, t) for t in ("q", "k", "v", "do"))

    def step():
        out, cache = rank_forward(ctx, q, k, v, masked=masked)
        g = rank_backward(ctx, cache, do)
        return out, g.dq, g.dk, g.dv

    eager = [t.clone() for t in step()]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        outs = step()
    for t in (q, k, v, do):
        t.mul_(1.0)  # same data; replay must reproduce eager bit for bit
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, outs):
        assert torch.equal(a, b)
    assert ctx.stats.allgather_launches >= 2
