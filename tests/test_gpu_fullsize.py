"""Parity at the BASELINE.json bench sizes (cfg2: unmasked N=128K, cfg3: masked
N=512K; B=1 H=16 d=128, bf16, one rank) through an N-independent property:
at sampled token positions s, the layer's outputs must equal the closed forms
    O_s  = q_s S_s,   dQ_s = dO_s S_s^T,   dK_s = v_s G_s^T,   dV_s = k_s G_s
with S_s = sum_{i<=s} k_i^T v_i and G_s = sum_{i>=s} q_i^T dO_i (masked;
every i for unmasked) — lasp2.py:168-203 / oracle.py:50-108 restated per row.
The states are formed here in float64 from the same bf16 inputs (block
partial sums, torch on the GPU: the f64 numpy oracle would take minutes at
this N), so the check is exact up to the kernels' bf16 roundings (SURVEY §8a
note P: normalised error <= 1e-2)."""
import pytest
import torch

from paper_2502_07563_b200.datagen import gen_slots_device
from paper_2502_07563_b200.lasp2 import ChunkedSequence, lasp2_iteration

pytestmark = pytest.mark.gpu

H, D = 16, 128
HEADS = (0, 7, 15)


def sample_rows(n: int) -> torch.Tensor:
    edges = [0, 1, 127, 128, 129, n // 2 - 1, n // 2, n - 129, n - 128, n - 2, n - 1]
    g = torch.Generator().manual_seed(n)
    return torch.unique(torch.cat([torch.tensor(edges), torch.randint(0, n, (37,), generator=g)])).cuda()


def inclusive_states(x: torch.Tensor, y: torch.Tensor, rows: torch.Tensor, masked: bool, suffix: bool,
                     blk: int = 4096) -> torch.Tensor:
    """[len(rows), d, d] f64: sum over i<=s (suffix: i>=s; unmasked: all i) of x_i^T y_i."""
    n, d = x.shape
    nb = (n + blk - 1) // blk
    parts = torch.stack([x[b * blk:(b + 1) * blk].T @ y[b * blk:(b + 1) * blk] for b in range(nb)])
    if not masked:
        return parts.sum(0).expand(len(rows), d, d)
    out = []
    for s in rows.tolist():
        b = s // blk
        if not suffix:
            acc = parts[:b].sum(0) + x[b * blk:s + 1].T @ y[b * blk:s + 1]
        else:
            acc = parts[b + 1:].sum(0) + x[s:(b + 1) * blk].T @ y[s:(b + 1) * blk]
        out.append(acc)
    return torch.stack(out)


@pytest.mark.parametrize("n,masked", [(131072, False), (524288, True)])
def test_bench_size_sampled_rows_match_closed_form(n, masked):
    q, k, v, do = (gen_slots_device(0, 1, H, n, D, t) for t in ("q", "k", "v", "do"))
    it = lasp2_iteration(ChunkedSequence(q, k, v, 1), do, masked)
    got = {"out": it.outputs[0], "dq": it.grads[0].dq, "dk": it.grads[0].dk, "dv": it.grads[0].dv}
    rows = sample_rows(n)
    for h in HEADS:
        qh, kh, vh, dh = (x[0, h].double() for x in (q, k, v, do))
        s_fw = inclusive_states(kh, vh, rows, masked, suffix=False)
        g_bw = inclusive_states(qh, dh, rows, masked, suffix=True)
        want = {
            "out": torch.einsum("rd,rde->re", qh[rows], s_fw),
            "dq": torch.einsum("rd,red->re", dh[rows], s_fw),
            "dk": torch.einsum("rd,red->re", vh[rows], g_bw),
            "dv": torch.einsum("rd,rde->re", kh[rows], g_bw),
        }
        for name, ref in want.items():
            g = got[name][0, h][rows].double()
            assert torch.isfinite(g).all(), name
            err = ((g - ref).abs().max() / ref.abs().max()).item()
            assert err <= 1e-2, (h, name, err)
