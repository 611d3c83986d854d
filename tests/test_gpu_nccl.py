"""The C ABI's NCCL wrappers (lasp2_state_allgather, lasp2h_kv_allgather,
lasp2h_grad_reduce_scatter) on a one-rank communicator, and
DistRankContext(native_collectives=True) — the rank programs' exchanges
through those wrappers — against torch.distributed's NCCL path and the
world-of-one context, bit for bit (one GPU: a world of one rank)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist

from paper_2502_07563_b200 import comm, lasp2, standard_sp
from paper_2502_07563_b200.datagen import gen_slots_device

pytestmark = pytest.mark.gpu


def test_nccl_comm_one_rank_wrappers():
    uid = comm.NcclComm.unique_id()
    assert len(uid) == 128
    c = comm.NcclComm(1, 0, uid)
    try:
        st = torch.randn(16, 128, 128, device="cuda")
        g = c.all_gather(st)
        torch.cuda.synchronize()
        assert g.shape == (1, 16, 128, 128) and torch.equal(g[0], st)
        k, v = (gen_slots_device(0, 1, 4, 256, 64, t) for t in ("k", "v"))
        kf, vf = c.all_gather_kv(k, v)
        torch.cuda.synchronize()
        assert torch.equal(kf[0], k) and torch.equal(vf[0], v)
        contrib = torch.randn(1, 2, 4, 256, 64, device="cuda", dtype=torch.float64)
        out = c.reduce_scatter(contrib)
        torch.cuda.synchronize()
        assert torch.equal(out, contrib[0])
        with pytest.raises(ValueError):
            c.reduce_scatter(torch.zeros(2, 3, device="cuda"))
    finally:
        c.close()


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_dist_native_collectives_match_torch_and_local():
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        native, plain, local = comm.DistRankContext(native_collectives=True), comm.DistRankContext(), \
            comm.LocalRankContext()
        assert native.nccl is not None and plain.nccl is None
        q, k, v, do = (gen_slots_device(0, 1, 4, 4096, 128, t) for t in ("q", "k", "v", "do"))
        for masked in (True, False):
            res = []
            for ctx in (native, plain, local):
                out, cache = lasp2.rank_forward(ctx, q, k, v, masked=masked)
                g = lasp2.rank_backward(ctx, cache, do)
                res.append([out, g.dq, g.dk, g.dv])
            torch.cuda.synchronize()
            for a, b, c in zip(*res):
                assert torch.equal(a, b) and torch.equal(a, c)
        res = []
        for ctx in (native, plain, local):
            out, cache = standard_sp._cp_forward_rank(ctx, q, k, v, True)
            g = standard_sp._cp_backward_rank(ctx, cache, do)
            res.append([out, g.dq, g.dk, g.dv])
        torch.cuda.synchronize()
        for a, b, c in zip(*res):
            assert torch.equal(a, b) and torch.equal(a, c)
        assert native.stats.allgather_launches == plain.stats.allgather_launches > 0
        assert native.stats.reduce_scatter_launches == plain.stats.reduce_scatter_launches == 1
        native.nccl.close()
    finally:
        dist.destroy_process_group()
