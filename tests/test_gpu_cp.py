"""LASP-2H softmax layers (AllGather K/V + causal softmax) on the GPU, mirroring
pkg/tests/test_standard_sp.py and acceptance criterion 6."""
import numpy as np
import pytest
import torch

from oracle import lasp_oracle as O
from paper_2502_07563_b200.lasp2 import ChunkedSequence
from paper_2502_07563_b200.standard_sp import cp_backward, cp_forward, cp_iteration

pytestmark = pytest.mark.gpu

CP_CASES = [(8, 4, 2, 1, 1, 0), (16, 8, 4, 1, 1, 0), (16, 4, 2, 1, 1, 0), (8, 4, 4, 2, 2, 3), (256, 32, 4, 1, 2, 1)]


def cat(xs):
    return torch.cat(list(xs), dim=2)


def to_np(t):
    return t.double().cpu().numpy()


def dev(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("case", CP_CASES)
def test_f64_matches_reference_fixtures(golden, case, causal):
    n, d, t, b, h, seed = case
    q, k, v, do = O.inputs(n, d, b, h, seed)
    it = cp_iteration(ChunkedSequence(q, k, v, t), do, causal)
    key = f"cp_{'c' if causal else 'n'}_{n}_{d}_{t}_{b}_{h}_{seed}"
    assert np.max(np.abs(to_np(cat(it.outputs)) - golden[key + "_out"])) <= 1e-12
    for name in ("dq", "dk", "dv"):
        got = to_np(cat(getattr(g, name) for g in it.grads))
        assert O.relative_error(got, golden[f"{key}_{name}"]) <= 1e-10, name
    # 2 all_gathers (K, V) + 1 reduce_scatter (dK/dV) = 3 steps (standard_sp.py:112-114)
    assert it.run.stats.communication_steps == 3
    assert it.run.stats.allgather_launches == 2 and it.run.stats.reduce_scatter_launches == 1


def test_zero_keys_causal_prefix_mean():
    q, _, v = O.qkv_slots(4, 1, 1, 8, 4)
    k = np.zeros_like(q)
    fwd = cp_forward(ChunkedSequence(q, k, v, 2), True)
    rows = v[0, 0]
    want = np.stack([rows[:i + 1].mean(axis=0) for i in range(8)])
    assert np.max(np.abs(to_np(cat(fwd.outputs))[0, 0] - want)) <= 1e-12


def test_forward_traffic_is_chunk_sized_keys_and_values():
    batch, heads, d, n, t = 2, 3, 4, 16, 4
    q, k, v, _ = O.inputs(n, d, batch, heads)
    fwd = cp_forward(ChunkedSequence(q, k, v, t))
    per_rank = 2 * batch * heads * (n // t) * d * 8
    for rank in range(t):
        assert fwd.run.rank_stats[rank].bytes_sent == per_rank


def test_iteration_traffic_adds_full_length_grads():
    batch, heads, d, n, t = 2, 1, 8, 16, 4
    q, k, v, do = O.inputs(n, d, batch, heads)
    it = cp_iteration(ChunkedSequence(q, k, v, t), do)
    per_rank = batch * heads * d * 8 * (2 * (n // t) + 2 * n)
    for rank in range(t):
        assert it.run.rank_stats[rank].bytes_sent == per_rank


def test_backward_rejects_wrong_caches():
    q, k, v, do = O.inputs(8, 4)
    seq = ChunkedSequence(q, k, v, 2)
    caches = cp_forward(seq, True).caches
    with pytest.raises(ValueError):
        cp_backward(seq, do, False, caches)
    with pytest.raises(ValueError):
        cp_backward(seq, do, True, caches[:1])


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.bfloat16, 1e-2)])
def test_low_precision_modes(dtype, tol):
    q, k, v, do = O.inputs(1024, 64, 1, 2, 5)
    if dtype == torch.bfloat16:
        q, k, v, do = (O.bf16_round(x) for x in (q, k, v, do))
    else:
        q, k, v, do = (x.astype(np.float32).astype(np.float64) for x in (q, k, v, do))
    ref = O.cp_full(q, k, v, do, 4, True)
    it = cp_iteration(ChunkedSequence(*(dev(x, dtype) for x in (q, k, v)), 4), dev(do, dtype), True)
    got = [to_np(cat(it.outputs))] + [to_np(cat(getattr(g, n) for g in it.grads)) for n in ("dq", "dk", "dv")]
    for name, g, r in zip(("out", "dq", "dk", "dv"), got, ref):
        assert O.normalized_error(g, r) <= tol, name


@pytest.mark.parametrize("t", [3, 4, 5, 8])
def test_balanced_schedule_f64_matches_oracle(t, monkeypatch):
    """Causal load balance (standard_sp.BALANCED): helpers compute leading key chunks of the
    upper ranks' queries; outputs / grads still match the reference math, with P2P sends."""
    import paper_2502_07563_b200.standard_sp as sp
    monkeypatch.setattr(sp, "BALANCED", True)
    n, d, b, h = 8 * t, 8, 1, 2
    q, k, v, do = O.inputs(n, d, b, h, 4)
    it = cp_iteration(ChunkedSequence(q, k, v, t), do, True)
    out, dq, dk, dv = O.cp_full(q, k, v, do, t, True)
    assert np.max(np.abs(to_np(cat(it.outputs)) - out)) <= 1e-12
    for name, ref in (("dq", dq), ("dk", dk), ("dv", dv)):
        assert O.relative_error(to_np(cat(getattr(g, name) for g in it.grads)), ref) <= 1e-10, name
    pairs = sum(1 for r in range(t) if sp._pairing(r, t, n // t, 1)[0] >= 0)
    assert it.run.stats.p2p_sends == 7 * pairs  # fwd: Q, O, lse; bwd: O, lse, dO, dQ
    assert it.run.stats.allgather_launches == 2 and it.run.stats.reduce_scatter_launches == 1


@pytest.mark.parametrize("t,c", [(4, 256), (8, 256), (4, 384)])
def test_balanced_schedule_bf16_matches_unbalanced(t, c, monkeypatch):
    """bf16: half-chunk offloads (c = 256) and offloads rounded down to 128-key blocks that
    start inside a chunk (c = 384: kv_start = 128) against the contiguous schedule."""
    import paper_2502_07563_b200.standard_sp as sp
    n, d, b, h = c * t, 128, 1, 2
    q, k, v, do = (O.bf16_round(x) for x in O.inputs(n, d, b, h, 5))
    seq = ChunkedSequence(*(torch.from_numpy(x).to("cuda", torch.bfloat16) for x in (q, k, v)), t)
    dod = torch.from_numpy(do).to("cuda", torch.bfloat16)
    plain = cp_iteration(seq, dod, True)
    monkeypatch.setattr(sp, "BALANCED", True)
    bal = cp_iteration(seq, dod, True)
    ref = O.cp_full(q, k, v, do, t, True)
    for got, want, r in zip([cat(bal.outputs)] + [cat(getattr(g, nm) for g in bal.grads) for nm in ("dq", "dk", "dv")],
                            [cat(plain.outputs)] + [cat(getattr(g, nm) for g in plain.grads)
                                                    for nm in ("dq", "dk", "dv")], ref):
        assert O.normalized_error(to_np(got), r) <= 1e-2
        assert O.normalized_error(to_np(got), to_np(want)) <= 1e-2


def test_pairing_balances_to_half_the_world():
    """Offloaded keys give every paired rank T/2 chunk-squares of causal work at even T."""
    import paper_2502_07563_b200.standard_sp as sp
    for world in (2, 4, 8):
        c = 1024
        cost = [(r + 0.5) * c * c for r in range(world)]
        for r in range(world):
            helper, guest, u = sp._pairing(r, world, c, 128)
            if helper >= 0:
                cost[r] -= u * c
                cost[helper] += u * c
        assert max(cost) == pytest.approx(world / 2 * c * c), (world, cost)
