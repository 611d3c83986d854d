"""Multi-process (gloo, world_size 2, CPU) coverage of the N>1 plumbing.

The per-rank LASP-2 / LASP-2H collective structure — one state all_gather per
pass, prefix/suffix folds of the rank-major gathered tensor, one
reduce_scatter of rank-major dK/dV contributions — runs through
DistRankContext exactly as under torchrun. Local math uses the oracle (CPU)
so the test checks the exchange layout and ledger, not the kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lasp_oracle as O
from paper_2502_07563_b200.comm import DistRankContext


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = DistRankContext()
        n, d, b, h = 32, 4, 1, 2
        q, k, v, do = O.inputs(n, d, b, h, seed=3)
        c = n // world
        sl = slice(rank * c, (rank + 1) * c)
        qc, kc, vc, dc = (torch.from_numpy(np.ascontiguousarray(x[:, :, sl])) for x in (q, k, v, do))
        t = ctx.sp_position
        # forward: M_t all_gather -> prefix fold -> intra + inter (lasp2.py:219-243)
        m_t = kc.transpose(-1, -2) @ vc
        gathered = ctx.all_gather(m_t.reshape(b * h * d, d)).view(world, b, h, d, d).numpy()
        m_prefix = O.prefix_sum_states(list(gathered), t)
        out = O.intra_forward_blocked(qc.numpy(), kc.numpy(), vc.numpy(), 4)
        if t > 0:
            out = out + qc.numpy() @ m_prefix
        # backward: dM all_gather (async) -> suffix fold (lasp2.py:270-285)
        g_t = qc.transpose(-1, -2) @ dc
        pending = ctx.all_gather_async(g_t.reshape(b * h * d, d))
        dq, dk, dv = O.intra_backward_blocked(qc.numpy(), kc.numpy(), vc.numpy(), dc.numpy(), 4)
        if t > 0:
            dq = dq + dc.numpy() @ np.swapaxes(m_prefix, -1, -2)
        g_all = pending.wait().view(world, b, h, d, d).numpy()
        if t < world - 1:
            dm = O.suffix_sum_states(list(g_all), t + 1)
            dk = dk + vc.numpy() @ np.swapaxes(dm, -1, -2)
            dv = dv + kc.numpy() @ dm
        # LASP-2H: rank-major contributions [T][2][...] -> one reduce_scatter
        contrib = torch.zeros((world, 2, b, h, c, d), dtype=torch.float64)
        contrib[:, 0] = torch.from_numpy(np.ascontiguousarray(
            np.stack(np.split(np.full((b, h, n, d), rank + 1.0), world, axis=2))))
        contrib[:, 1] = 10.0 * (rank + 1.0)
        mine = ctx.reduce_scatter(contrib)
        results[rank] = dict(out=out, dq=dq, dk=dk, dv=dv, rs=mine.numpy(),
                             stats=(ctx.stats.allgather_launches, ctx.stats.reduce_scatter_launches,
                                    ctx.stats.bytes_sent))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_lasp2_exchange_matches_oracle():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    q, k, v, do = O.inputs(32, 4, 1, 2, seed=3)
    out, dq, dk, dv = O.lasp2_full(q, k, v, do, world, True, bc=4)
    c = 16
    for r in range(world):
        sl = slice(r * c, (r + 1) * c)
        res = results[r]
        assert np.max(np.abs(res["out"] - out[:, :, sl])) <= 1e-12
        for name, ref in (("dq", dq), ("dk", dk), ("dv", dv)):
            assert O.relative_error(res[name], ref[:, :, sl]) <= 1e-12
        assert np.allclose(res["rs"][0], 3.0) and np.allclose(res["rs"][1], 30.0)
        ag, rs, nbytes = res["stats"]
        assert ag == 2 and rs == 1  # 2 state all_gathers per iteration (+1 LASP-2H reduce_scatter)
        state_bytes = 1 * 2 * 4 * 4 * 8
        assert nbytes == 2 * state_bytes + world * 2 * 1 * 2 * c * 4 * 8


def _ring_worker(rank, world, port, results):
    """LASP-1 ring plumbing (lasp1.py:43-72, 82-107) through DistRankContext.send/recv."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = DistRankContext()
        n, d, b, h = 24, 4, 1, 2
        q, k, v, do = O.inputs(n, d, b, h, seed=4)
        c = n // world
        sl = slice(rank * c, (rank + 1) * c)
        kc, vc, qc, dc = (torch.from_numpy(np.ascontiguousarray(x[:, :, sl])) for x in (k, v, q, do))
        r, peers = ctx.sp_position, ctx.sp_peers
        own = (kc.transpose(-1, -2) @ vc).reshape(b * h * d, d)
        if r == 0:
            prefix, upd = torch.zeros_like(own), own.clone()
        else:
            prefix = ctx.recv(peers[r - 1], tag="state", like=own)
            upd = prefix.clone()
            upd += own
        if r < world - 1:
            ctx.send(peers[r + 1], upd, tag="state")
        g = (qc.transpose(-1, -2) @ dc).reshape(b * h * d, d)
        if r < world - 1:
            suffix = ctx.recv(peers[r + 1], tag="state_grad", like=g)
            gup = suffix.clone()
            gup += g
        else:
            suffix, gup = torch.zeros_like(g), g.clone()
        if r > 0:
            ctx.send(peers[r - 1], gup, tag="state_grad")
        results[rank] = dict(prefix=prefix.numpy(), suffix=suffix.numpy(), through=upd.numpy(),
                             stats=(ctx.stats.p2p_sends, ctx.stats.p2p_recvs, ctx.stats.bytes_sent))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_three_rank_gloo_ring_send_recv():
    world = 3
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_ring_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    q, k, v, do = O.inputs(24, 4, 1, 2, seed=4)
    c = 8
    chunk = lambda x, i: x[:, :, i * c:(i + 1) * c]  # noqa: E731
    states = [(np.swapaxes(chunk(k, i), -1, -2) @ chunk(v, i)).reshape(8, 4) for i in range(world)]
    grads = [(np.swapaxes(chunk(q, i), -1, -2) @ chunk(do, i)).reshape(8, 4) for i in range(world)]
    for r in range(world):
        res = results[r]
        assert np.allclose(res["prefix"], O.prefix_sum_states(states, r), rtol=0, atol=1e-12)
        assert np.allclose(res["suffix"], O.suffix_sum_states(grads, r + 1), rtol=0, atol=1e-12)
        sends, recvs, nbytes = res["stats"]
        want = (r < world - 1) + (r > 0)  # one hop each way except at the ends
        assert sends == recvs == want and nbytes == want * 8 * 4 * 8
    assert np.allclose(results[world - 1]["through"], O.sum_states(states), rtol=0, atol=1e-12)


def _owners_worker(rank, world, port, counts, results):
    """LASP-2H dK/dV reduction without causal zeros (DistRankContext.reduce_to_owners)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = DistRankContext()
        # rank t's contribution to owner r: 10**t + r (exact in f64), shape (2, 3)
        contrib = torch.stack([torch.full((2, 3), 10.0 ** rank + r, dtype=torch.float64)
                               for r in range(counts[rank])])
        mine = ctx.reduce_to_owners(contrib, counts, tag="dkv")
        results[rank] = dict(mine=mine.numpy(), stats=(ctx.stats.reduce_scatter_launches, ctx.stats.bytes_sent,
                                                       ctx.stats.p2p_sends))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("counts", [[1, 2, 3], [1, 3, 3], [3, 3, 3]])
def test_three_rank_gloo_reduce_to_owners(counts):
    """Causal counts (t + 1), a balanced helper holding a later chunk, and the full
    (non-causal) case: owner r gets the ascending-rank sum of every rank with counts[t] > r,
    one reduce_scatter launch in the ledger with the bytes actually sent."""
    world = 3
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_owners_worker, args=(world, _free_port(), counts, results), nprocs=world, join=True)
    for r in range(world):
        want = sum(10.0 ** t + r for t in range(world) if counts[t] > r)
        assert np.array_equal(results[r]["mine"], np.full((2, 3), want))
        rs, nbytes, p2p = results[r]["stats"]
        sent = sum(1 for o in range(counts[r]) if o != r)
        assert rs == 1 and p2p == 0 and nbytes == sent * 6 * 8
