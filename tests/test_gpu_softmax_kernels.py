"""tcgen05 flash-attention kernels for LASP-2H against fp64 torch math, with the
rank-major full-length K/V layout the all_gather produces and global causal
offsets (oracle.py:111-158 semantics)."""
import math

import pytest
import torch

from paper_2502_07563_b200 import ops

pytestmark = pytest.mark.gpu


def rand(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return ((torch.rand(shape, generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * scale).to(torch.bfloat16)


def nerr(got, ref):
    got, ref = got.double(), ref.double()
    return ((got - ref).abs().max() / ref.abs().max()).item()


def reference(q, kfull, vfull, do, causal, row_offset):
    """fp64 softmax attention of q rows [row_offset, ...) against plain [B,H,N,d] K/V."""
    qd, kd, vd = q.double(), kfull.double(), vfull.double()
    d = q.shape[-1]
    s = qd @ kd.transpose(-1, -2) / math.sqrt(d)
    if causal:
        rows = row_offset + torch.arange(q.shape[2], device=q.device)[:, None]
        cols = torch.arange(kfull.shape[2], device=q.device)[None, :]
        s = s.masked_fill(cols > rows, float("-inf"))
    p = torch.softmax(s, dim=-1)
    o = p @ vd
    lse = torch.logsumexp(s, dim=-1)
    dod = do.double()
    dv = p.transpose(-1, -2) @ dod
    dp = dod @ vd.transpose(-1, -2)
    ds = p * (dp - (dp * p).sum(-1, keepdim=True))
    dq = ds @ kd / math.sqrt(d)
    dk = ds.transpose(-1, -2) @ qd / math.sqrt(d)
    return o, lse, dq, dk, dv


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("b,h,t,c,d,rank", [(1, 2, 4, 256, 128, 2), (1, 1, 2, 384, 64, 1), (2, 1, 1, 512, 128, 0),
                                            (1, 2, 8, 128, 128, 7), (1, 1, 3, 256, 32, 0)])
def test_softmax_fwd_bwd_rank_major(causal, b, h, t, c, d, rank):
    n = t * c
    kf = rand((t, b, h, c, d), 1)  # rank-major, as all_gather_into_tensor writes it
    vf = rand((t, b, h, c, d), 2)
    q = rand((b, h, c, d), 3)
    do = rand((b, h, c, d), 4)
    row_offset = rank * c
    plain_k = kf.permute(1, 2, 0, 3, 4).reshape(b, h, n, d)
    plain_v = vf.permute(1, 2, 0, 3, 4).reshape(b, h, n, d)
    ro, rlse, rdq, rdk, rdv = reference(q, plain_k, plain_v, do, causal, row_offset)
    per = b * h * c * d
    out, lse = ops.softmax_forward(q, kf, vf, causal, row_offset, kv_tokens=n, kv_chunk=c, kv_rank_stride=per)
    assert nerr(out, ro) <= 1e-2
    assert (lse.double() - rlse).abs().max().item() <= 2e-2
    grads = torch.empty((t, 2, b, h, c, d), dtype=torch.float32, device="cuda")
    dq = ops.softmax_backward(q, kf, vf, out, lse, do, causal, row_offset, kv_tokens=n, kv_chunk=c,
                              kv_rank_stride=per, grads=grads, grad_rank_stride=2 * per, dv_offset=per)
    dk = grads[:, 0].permute(1, 2, 0, 3, 4).reshape(b, h, n, d)
    dv = grads[:, 1].permute(1, 2, 0, 3, 4).reshape(b, h, n, d)
    assert nerr(dq, rdq) <= 1e-2
    assert nerr(dk, rdk) <= 1e-2
    assert nerr(dv, rdv) <= 1e-2
    if causal:  # keys after this rank's last query get exactly zero contribution
        last = row_offset + c
        if last < n:
            assert torch.count_nonzero(dk[:, :, last:]) == 0 and torch.count_nonzero(dv[:, :, last:]) == 0


def test_softmax_plain_layout_ragged_queries():
    b, h, n, d = 1, 2, 640, 128
    k, v = rand((b, h, n, d), 5), rand((b, h, n, d), 6)
    q, do = rand((b, h, 200, d), 7), rand((b, h, 200, d), 8)
    ro, rlse, rdq, rdk, rdv = reference(q, k, v, do, True, 300)
    out, lse = ops.softmax_forward(q, k, v, True, 300, kv_tokens=n, kv_chunk=n, kv_rank_stride=0)
    assert nerr(out, ro) <= 1e-2
    grads = torch.empty((1, 2, b, h, n, d), dtype=torch.float32, device="cuda")
    per = b * h * n * d
    dq = ops.softmax_backward(q, k, v, out, lse, do, True, 300, kv_tokens=n, kv_chunk=n, kv_rank_stride=0,
                              grads=grads, grad_rank_stride=0, dv_offset=per)
    assert nerr(dq, rdq) <= 1e-2
    assert nerr(grads[0, 0], rdk) <= 1e-2 and nerr(grads[0, 1], rdv) <= 1e-2
