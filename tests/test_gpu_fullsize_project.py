"""The hybrid stack's projections (SURVEY §8f.1; reference hybrid.py:136-151, :216-231) on the path's
own kernels at the LASP-2H config size (cfg4: B=1, H=16, N=256K, d=128, bf16): lasp2_project's
X W, X W^T and the three-term dX = dQ W_Q^T + dK W_K^T + dV W_V^T (one accumulator, one rounding)
against float64 closed forms on sampled token rows of every head, and the weight gradient
X^T dY (segment contractions + ordered fold, hybrid.py's path) against a float64 sum."""
import pytest
import torch

from paper_2502_07563_b200 import ops
from paper_2502_07563_b200.datagen import gen_slots_device

pytestmark = pytest.mark.gpu

B, H, N, D = 1, 16, 262144, 128


def _rows():
    g = torch.Generator().manual_seed(5)
    edge = [0, 1, 127, 128, N // 2, N - 129, N - 128, N - 1]
    return torch.unique(torch.cat([torch.tensor(edge), torch.randint(0, N, (40,), generator=g)])).cuda()


def _w(seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn((D, D), generator=g, device="cuda") / D ** 0.5).contiguous()


def _nerr(got, ref):
    return ((got.double() - ref).abs().max() / ref.abs().max()).item()


def test_projections_at_cfg4_size():
    xs = [gen_slots_device(0, B, H, N, D, t) for t in ("x", "dq", "dk")]
    ws = [_w(s) for s in (1, 2, 3)]
    rows = _rows()
    x = xs[0]
    for transpose in (False, True):
        out = ops.project([x], [ws[0]], transpose=transpose)
        w = ws[0].double().T if transpose else ws[0].double()
        ref = x[0][:, rows].double() @ w
        assert _nerr(out[0][:, rows], ref) <= 1e-2
    out3 = ops.project(xs, ws, transpose=True)
    ref3 = sum(xi[0][:, rows].double() @ wi.double().T for xi, wi in zip(xs, ws))
    assert _nerr(out3[0][:, rows], ref3) <= 1e-2
    # accumulate onto an existing output
    base = ops.project([x], [ws[1]])
    acc = ops.project([x], [ws[2]], out=base.clone(), accumulate=True)
    ref_acc = base[0][:, rows].double() + x[0][:, rows].double() @ ws[2].double()
    assert _nerr(acc[0][:, rows], ref_acc) <= 1e-2


def test_weight_gradient_at_cfg4_size():
    x, dy = (gen_slots_device(0, B, H, N, D, t) for t in ("x", "dy"))
    nseg = ops.num_segments(x)
    seg = ops.segment_states(x, dy, nseg)                      # [B, H, nseg, D, D] fp32: X_g^T dY_g
    dw = ops.sum_states(seg.reshape(B * H * nseg, D, D))      # ordered fold over every slot and segment
    ref = torch.zeros((D, D), dtype=torch.float64, device="cuda")
    for h in range(H):
        for lo in range(0, N, 65536):
            ref += x[0, h, lo:lo + 65536].double().T @ dy[0, h, lo:lo + 65536].double()
    assert _nerr(dw, ref) <= 1e-3
