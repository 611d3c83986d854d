"""The unmasked world kernels with the state exchange fused in (lasp2_nomask_forward_x /
lasp2_nomask_backward_x): one launch per direction does phase 1, stores this rank's state into
every rank's receive half, waits for every rank's flag, folds the full sum and runs phase 2.

One process drives rank `rank` of a T-rank exchange whose other ranks are already complete:
their receive slots and flags are filled in advance (and their acks set), so the kernel's
own stores, flag release, wait, ordered fold, acknowledgement and epoch advance are checked
against the all_gather path (phase 1, lasp2_fold_states FULL, phase 2) bit for bit, over
several epochs (both receive halves). The cross-process run is tests/test_gpu_multiprocess.py."""
import pytest
import torch

from paper_2502_07563_b200 import ops
from paper_2502_07563_b200.comm import PeerExchange, _ptr_table
from paper_2502_07563_b200.datagen import gen_slots_device

pytestmark = pytest.mark.gpu

FAR = 1 << 62  # "already arrived" for the ranks this process does not run


def _world(rank: int, nranks: int, like: torch.Tensor, others: torch.Tensor):
    dev = like.device
    recv = [torch.zeros((2, nranks, *like.shape), dtype=like.dtype, device=dev) for _ in range(nranks)]
    flags = [torch.zeros(nranks, dtype=torch.int64, device=dev) for _ in range(nranks)]
    acks = [torch.zeros(nranks, dtype=torch.int64, device=dev) for _ in range(nranks)]
    for r in range(nranks):
        if r != rank:
            recv[rank][:, r] = others[r]  # both halves: rank r's state of every epoch
            flags[rank][r] = FAR
            acks[rank][r] = FAR
    done = torch.zeros(1, dtype=torch.int32, device=dev)
    tables = [_ptr_table(x, dev) for x in (recv, flags, acks)]
    torch.cuda.synchronize()
    return PeerExchange(rank, nranks, recv[rank], flags[rank], acks[rank], done, *tables), recv, flags, acks


@pytest.mark.parametrize("shape,rank,nranks", [((1, 16, 16384, 128), 7, 8), ((2, 3, 2000, 64), 1, 4),
                                               ((1, 2, 256, 128), 0, 1)])
def test_fused_flat_exchange_matches_allgather_path_bitwise(shape, rank, nranks):
    b, h, n, d = shape
    q, k, v, do = (gen_slots_device(0, b, h, n, d, t, row_offset=rank * n) for t in ("q", "k", "v", "do"))
    g = torch.Generator(device="cuda").manual_seed(rank)
    others = torch.randn((nranks, b, h, d, d), generator=g, device="cuda") * 40.0
    dothers = torch.randn((nranks, b, h, d, d), generator=g, device="cuda") * 40.0
    m_like = torch.empty((b, h, d, d), dtype=torch.float32, device="cuda")
    fx, recv_f, flags_f, _ = _world(rank, nranks, m_like, others)
    bx, recv_b, flags_b, _ = _world(rank, nranks, m_like, dothers)
    # the all_gather path for the same inputs
    m_t = ops.nomask_forward_phase(q, k, v, torch.empty_like(m_like), 1)
    gathered = others.clone()
    gathered[rank] = m_t
    m_ref = ops.sum_states(gathered)
    out_ref = ops.nomask_forward_phase(q, k, v, m_ref.contiguous(), 2)
    dq_ref, dm_t = ops.nomask_backward_phase1(q, do, m_ref.contiguous())
    dgathered = dothers.clone()
    dgathered[rank] = dm_t
    dm_ref = ops.sum_states(dgathered)
    dk_ref, dv_ref = ops.nomask_backward_phase2(v, k, dm_ref)
    for epoch in (1, 2, 3):  # both receive halves, and back-pressure on the own ack of epoch - 2
        out, m_full = ops.nomask_forward_x(q, k, v, fx)
        dq, dk, dv = ops.nomask_backward_x(q, k, v, do, m_full, bx)
        torch.cuda.synchronize()
        assert int(fx.ep.item()) == epoch and int(bx.ep.item()) == epoch
        assert torch.equal(m_full, m_ref) and torch.equal(out, out_ref)
        assert torch.equal(dq, dq_ref) and torch.equal(dk, dk_ref) and torch.equal(dv, dv_ref)
        for r in range(nranks):  # this rank's state landed in every rank's half of this epoch, flags released
            assert torch.equal(recv_f[r][epoch & 1, rank], m_t) and torch.equal(recv_b[r][epoch & 1, rank], dm_t)
            assert int(flags_f[r][rank].item()) == epoch and int(flags_b[r][rank].item()) == epoch
        assert int(fx.acks[rank].item()) == epoch  # acknowledged to itself like to every writer
