"""LASP-1 ring baseline on the GPU (reference pkg/tests/test_lasp1.py): the ring
drivers against the reference's own lasp1_iteration outputs in f64, against
the oracle in bf16, plus the ring's ledger, hop payloads and trace order."""
import importlib.util
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import lasp_oracle as O
from paper_2502_07563_b200.lasp1 import (lasp1_backward_masked, lasp1_backward_nomask, lasp1_forward_masked,
                                         lasp1_forward_nomask, lasp1_iteration)
from paper_2502_07563_b200.lasp2 import ChunkedSequence, lasp2_iteration

pytestmark = pytest.mark.gpu

_spec = importlib.util.spec_from_file_location("make_golden", Path(__file__).parent / "golden" / "make_golden.py")
_mg = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mg)
LASP1_CASES = _mg.LASP1_CASES


def cat(xs):
    return torch.cat(list(xs), dim=2).double().cpu().numpy()


def grads(it):
    return [cat(getattr(g, nm) for g in it.grads) for nm in ("dq", "dk", "dv")]


@pytest.mark.parametrize("masked", [True, False])
@pytest.mark.parametrize("case", LASP1_CASES)
def test_f64_ring_matches_reference(lasp1_golden, case, masked):
    n, d, t, b, h, seed = case
    q, k, v, do = O.inputs(n, d, b, h, seed)
    it = lasp1_iteration(ChunkedSequence(q, k, v, t), do, masked)
    key = f"l1_{'m' if masked else 'u'}_{n}_{d}_{t}_{b}_{h}_{seed}"
    assert np.max(np.abs(cat(it.outputs) - lasp1_golden[key + "_out"])) <= 1e-10
    for got, nm in zip(grads(it), ("dq", "dk", "dv")):
        assert O.relative_error(got, lasp1_golden[f"{key}_{nm}"]) <= 1e-12, nm
    through = it.caches[-1].state_through.double().cpu().numpy()
    assert O.relative_error(through, lasp1_golden[key + "_through"]) <= 1e-12
    st = it.run.stats
    assert st.p2p_sends == st.communication_steps == 2 * (t - 1)
    assert st.allgather_launches == 0 and st.bytes_sent == 2 * (t - 1) * b * h * d * d * 8


@pytest.mark.parametrize("n,t", [(4096, 2), (8192, 4)])
def test_bf16_ring_matches_oracle_and_allgather_method(n, t):
    d, b, h = 128, 1, 2
    q, k, v, do = (O.bf16_round(x) for x in O.inputs(n, d, b, h, 5))
    dev = lambda x: torch.from_numpy(x).to("cuda", torch.bfloat16)  # noqa: E731
    seq = ChunkedSequence(dev(q), dev(k), dev(v), t)
    ring = lasp1_iteration(seq, dev(do), True)
    ref = O.lasp2_full(q, k, v, do, t, True)
    got = [cat(ring.outputs)] + grads(ring)
    for g, r, nm in zip(got, ref, ("out", "dq", "dk", "dv")):
        assert O.normalized_error(g, r) <= 1e-2, nm
    gather = lasp2_iteration(seq, dev(do), True)
    for g, r in zip(got, [cat(gather.outputs)] + grads(gather)):
        assert O.normalized_error(g, r) <= 1e-2
    assert ring.run.stats.p2p_sends == 2 * (t - 1) and gather.run.stats.allgather_launches == 2


def test_single_chunk_needs_no_comm():
    q, k, v, do = O.inputs(8, 4)
    it = lasp1_iteration(ChunkedSequence(q, k, v, 1), do, True)
    assert it.run.stats.communication_steps == 0 and it.run.stats.bytes_sent == 0


def test_ring_state_bytes_per_hop_and_forward_steps():
    q, k, v, _ = O.inputs(16, 4, 2, 3)
    fwd = lasp1_forward_masked(ChunkedSequence(q, k, v, 4))
    assert fwd.run.stats.bytes_sent == 3 * (2 * 3 * 4 * 4 * 8)
    assert fwd.run.stats.p2p_sends == 3 and fwd.run.stats.allgather_launches == 0


def test_unmasked_rank0_zero_and_last_rank_zero_kv_grads():
    q, k, v, do = O.inputs(16, 4, seed=3)
    seq = ChunkedSequence(q, k, v, 4)
    fwd = lasp1_forward_nomask(seq)
    assert not fwd.outputs[0].any()
    bwd = lasp1_backward_nomask(seq, do, fwd.caches)
    assert not bwd.grads[-1].dk.any() and not bwd.grads[-1].dv.any()
    out, dq, dk, dv = O.lasp1_nomask_full(q, k, v, do, 4)
    assert np.max(np.abs(cat(fwd.outputs) - out)) <= 1e-12
    assert O.relative_error(cat(g.dq for g in bwd.grads), dq) <= 1e-12


def test_masked_zero_upstream_gives_zero_grads():
    q, k, v, do = O.inputs(8, 4)
    it = lasp1_iteration(ChunkedSequence(q, k, v, 4), np.zeros_like(do), True)
    for g in grads(it):
        assert not g.any()


def test_ring_order_in_trace():
    q, k, v, _ = O.inputs(8, 4)
    fwd = lasp1_forward_masked(ChunkedSequence(q, k, v, 4))
    sends = {ev.rank: ev.seq for ev in fwd.run.trace if ev.kind == "send"}
    inters = {ev.rank: ev.seq for ev in fwd.run.trace if ev.kind == "inter_start"}
    assert sorted(sends) == [0, 1, 2] and sorted(inters) == [1, 2, 3]
    for rank in (1, 2, 3):  # a rank folds its prefix only after the previous rank sent it
        assert inters[rank] > sends[rank - 1]


def test_backward_rejects_wrong_caches():
    q, k, v, do = O.inputs(8, 4)
    seq = ChunkedSequence(q, k, v, 2)
    caches = lasp1_forward_nomask(seq).caches
    with pytest.raises(ValueError):
        lasp1_backward_masked(seq, do, caches)
    with pytest.raises(ValueError):
        lasp1_backward_nomask(seq, do, caches[:1])
