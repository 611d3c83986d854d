"""LASP-2H parity at the cfg4 per-rank size (BASELINE.json configs[3]: N=256K,
W=8, C=32K, H=16, d=128, bf16): the softmax kernels of rank t against keys /
values in the rank-major all_gather layout, checked at sampled rows through
the closed forms of oracle.py:111-158 evaluated in float64 on the same bf16
inputs (the f64 numpy oracle would take hours at this size):
    o_s = softmax(q_s K^T / sqrt(d), causal) V,   lse_s = logsumexp(...)
    dq_s = sum_j P_sj (dP_sj - D_s) k_j / sqrt(d)          (dP_sj = do_s . v_j)
    dk_j = sum_s P_sj (dP_sj - D_s) q_s / sqrt(d),  dv_j = sum_s P_sj do_s
(dk/dv: this rank's contributions, the reduce-scatter input). The backward's
reference uses the forward's lse and D_s = do_s . o_s (equal to
rowsum(P o dP) in exact arithmetic), so each pass is checked on its own.
Tolerance: normalised error <= 1e-2 (SURVEY §8a note P), lse absolute 1e-3."""
import math

import pytest
import torch

from paper_2502_07563_b200 import ops
from paper_2502_07563_b200.datagen import gen_slots_device

pytestmark = pytest.mark.gpu

W, N, H, D = 8, 262144, 16, 128
C = N // W
HEADS = (0, 9)


def _nerr(got: torch.Tensor, ref: torch.Tensor) -> float:
    return ((got.double() - ref).abs().max() / ref.abs().max()).item()


@pytest.mark.parametrize("t", [7, 2])
def test_cfg4_rank_sampled_rows_match_closed_forms(t):
    q, do = (gen_slots_device(0, 1, H, C, D, tag, row_offset=t * C) for tag in ("q", "do"))
    kf = torch.stack([gen_slots_device(0, 1, H, C, D, "k", row_offset=r * C).reshape(H * C, D) for r in range(W)])
    vf = torch.stack([gen_slots_device(0, 1, H, C, D, "v", row_offset=r * C).reshape(H * C, D) for r in range(W)])
    stride = H * C * D
    out, lse = ops.softmax_forward(q, kf, vf, True, t * C, kv_tokens=N, kv_chunk=C, kv_rank_stride=stride)
    grads = torch.zeros((W, 2, 1, H, C, D), dtype=torch.float32, device="cuda")
    dq = ops.softmax_backward(q, kf, vf, out, lse, do, True, t * C, N, C, stride, grads, 2 * stride, stride)
    torch.cuda.synchronize()
    scale = 1.0 / math.sqrt(D)
    g = torch.Generator().manual_seed(t)
    rows = torch.unique(torch.cat([torch.tensor([0, 1, 127, 128, C // 2, C - 1]),
                                   torch.randint(0, C, (26,), generator=g)])).cuda()
    keys = torch.unique(torch.cat([torch.tensor([0, C - 1, t * C, t * C + 5, (t + 1) * C - 1]),
                                   torch.randint(0, (t + 1) * C, (19,), generator=g)])).cuda()
    for h in HEADS:
        kh = kf[:, h * C:(h + 1) * C].reshape(N, D).double()   # global key order
        vh = vf[:, h * C:(h + 1) * C].reshape(N, D).double()
        qh, dh, oh = q[0, h].double(), do[0, h].double(), out[0, h].double()
        lse_h = lse[0, h].double()
        # forward and dQ at sampled query rows
        o_ref, dq_ref, lse_ref = [], [], []
        for s in rows.tolist():
            gq = t * C + s
            sc = (kh[:gq + 1] @ qh[s]) * scale
            m = sc.max()
            p = torch.exp(sc - m)
            l = p.sum()
            p = p / l
            lse_ref.append(m + torch.log(l))
            o_ref.append(p @ vh[:gq + 1])
            dp = vh[:gq + 1] @ dh[s]
            delta = (dh[s] * oh[s]).sum()
            dq_ref.append(((p * (dp - delta)) @ kh[:gq + 1]) * scale)
        assert _nerr(out[0, h][rows], torch.stack(o_ref)) <= 1e-2, (t, h, "out")
        assert (lse_h[rows] - torch.stack(lse_ref)).abs().max().item() <= 1e-3, (t, h, "lse")
        assert _nerr(dq[0, h][rows], torch.stack(dq_ref)) <= 1e-2, (t, h, "dq")
        # this rank's dK / dV contributions at sampled keys
        gq_all = t * C + torch.arange(C, device="cuda")
        delta_all = (dh * oh).sum(-1)
        dk_ref, dv_ref = [], []
        for j in keys.tolist():
            vis = (gq_all >= j).double()
            p = torch.exp((qh @ kh[j]) * scale - lse_h) * vis
            ds = p * (dh @ vh[j] - delta_all)
            dk_ref.append((ds @ qh) * scale)
            dv_ref.append(p @ dh)
        rk, ck = keys // C, keys % C
        assert _nerr(grads[rk, 0, 0, h, ck], torch.stack(dk_ref)) <= 1e-2, (t, h, "dk")
        assert _nerr(grads[rk, 1, 0, h, ck], torch.stack(dv_ref)) <= 1e-2, (t, h, "dv")
