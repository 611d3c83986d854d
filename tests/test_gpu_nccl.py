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
        for name, a, b, c in zip(("out", "dq", "dk", "dv"), *res):
            if name == "dq":  # fp32 reduce-adds of the key blocks in a timing-dependent order: ~1 bf16 ulp
                for x in (b, c):
                    assert ((a.float() - x.float()).abs().max() / a.float().abs().max()).item() <= 1e-2
            else:
                assert torch.equal(a, b) and torch.equal(a, c), name
        assert native.stats.allgather_launches == plain.stats.allgather_launches > 0
        assert native.stats.reduce_scatter_launches == plain.stats.reduce_scatter_launches == 1
        native.nccl.close()
    finally:
        dist.destroy_process_group()


def test_integration_stub_unmasked_rank_through_the_c_abi():
    """INTEGRATION.md's T-rank unmasked forward through raw C-ABI calls (phase 1, the
    NCCL state AllGather wrapper, the full fold, phase 2) on a one-rank world equals
    the world-of-one persistent launch bit for bit."""
    import ctypes

    from paper_2502_07563_b200 import _lib, ops

    lib = _lib.load()
    stream = torch.cuda.current_stream().cuda_stream
    q, k, v = (gen_slots_device(0, 1, 4, 4096, 128, t) for t in ("q", "k", "v"))
    b, h, c, d = q.shape
    ws = ops.local_workspace(q)
    uid = ctypes.create_string_buffer(128)
    assert lib.lasp2_nccl_unique_id(ctypes.addressof(uid)) == 0
    handle = ctypes.c_void_p()
    assert lib.lasp2_nccl_comm_init(ctypes.addressof(handle), 1, ctypes.addressof(uid), 0) == 0
    try:
        m_t = torch.empty((b, h, d, d), dtype=torch.float32, device="cuda")
        assert lib.lasp2_nomask_forward_phase(_lib.BF16, None, k.data_ptr(), v.data_ptr(), None, m_t.data_ptr(),
                                              ws.data_ptr(), ws.numel(), b * h, c, d, 1, stream) == 0
        gathered = torch.empty((1, b, h, d, d), dtype=torch.float32, device="cuda")
        assert lib.lasp2_state_allgather(handle.value, _lib.F32, m_t.data_ptr(), gathered.data_ptr(), m_t.numel(),
                                         stream) == 0
        m_full = torch.empty_like(m_t)
        assert lib.lasp2_fold_states(_lib.F32, gathered.data_ptr(), m_full.data_ptr(), 1, m_full.numel(), 2, 0,
                                     stream) == 0
        out = torch.empty_like(q)
        assert lib.lasp2_nomask_forward_phase(_lib.BF16, q.data_ptr(), None, None, out.data_ptr(),
                                              m_full.data_ptr(), ws.data_ptr(), ws.numel(), b * h, c, d, 2,
                                              stream) == 0
        ref_out, ref_m = ops.nomask_forward_local(q, k, v)
        torch.cuda.synchronize()
        assert torch.equal(out, ref_out) and torch.equal(m_full, ref_m)
    finally:
        lib.lasp2_nccl_comm_destroy(handle.value)
