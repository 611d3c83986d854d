"""LASP-2 layer parity on the GPU through the C ABI, mirroring the reference
suite (pkg/tests/test_lasp2.py, test_acceptance.py c1/c2/c5/c8).

* float64 inputs run the validation kernels and must meet the reference's own
  tolerances against the reference's outputs (golden fixtures): forward
  max-abs 1e-10, gradients relative_error 1e-12 (test_lasp2.py:17-19).
* float32 (fp32 validation mode): normalised error <= 1e-4.
* bfloat16 (tcgen05 fast path): normalised error <= 1e-2 against the f64
  oracle evaluated on the same bf16-rounded inputs (SURVEY §8a note P).
"""
import numpy as np
import pytest
import torch

from oracle import lasp_oracle as O
from paper_2502_07563_b200 import comm
from paper_2502_07563_b200.lasp2 import (ActivationCache, ChunkedSequence, intra_backward, intra_forward,
                                         lasp2_backward_masked, lasp2_backward_nomask, lasp2_forward_masked,
                                         lasp2_forward_nomask, lasp2_iteration, lasp2_overlap_schedule)

pytestmark = pytest.mark.gpu

LASP_CASES = [(8, 4, 1, 1, 1, 0), (8, 4, 2, 1, 1, 0), (16, 8, 4, 1, 1, 0), (16, 4, 8, 1, 1, 0),
              (64, 16, 4, 1, 1, 0), (256, 16, 8, 1, 1, 0), (256, 4, 2, 1, 1, 0), (8, 4, 4, 2, 3, 5),
              (256, 32, 4, 1, 2, 7)]


def cat(xs):
    return torch.cat(list(xs), dim=2)


def to_np(t):
    return t.double().cpu().numpy()


def grads_np(it):
    return [to_np(cat(getattr(g, n) for g in it.grads)) for n in ("dq", "dk", "dv")]


def dev(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


@pytest.mark.parametrize("masked", [True, False])
@pytest.mark.parametrize("case", LASP_CASES)
def test_f64_matches_reference_fixtures(golden, case, masked):
    n, d, t, b, h, seed = case
    q, k, v, do = O.inputs(n, d, b, h, seed)
    it = lasp2_iteration(ChunkedSequence(q, k, v, t), do, masked)
    key = f"lasp2_{'m' if masked else 'u'}_{n}_{d}_{t}_{b}_{h}_{seed}"
    assert np.max(np.abs(to_np(cat(it.outputs)) - golden[key + "_out"])) <= 1e-10
    for name, g in zip(("dq", "dk", "dv"), grads_np(it)):
        assert O.relative_error(g, golden[f"{key}_{name}"]) <= 1e-12, name
    launches, nbytes = golden[key + "_launches"]
    assert it.run.stats.allgather_launches == launches == 2
    assert it.run.stats.bytes_sent == nbytes  # B*H*d^2*8 per rank per launch (costmodel.py:56-58)


def test_f64_backward_matches_finite_difference():
    q, k, v, do = O.inputs(8, 4, seed=3)
    for masked in (True, False):
        it = lasp2_iteration(ChunkedSequence(q, k, v, 2), do, masked)
        got = grads_np(it)
        for i in range(3):
            def loss(x, i=i):
                parts = [q, k, v]
                parts[i] = x
                out = np.stack([O.linear_attn_serial(parts[0][0, 0], parts[1][0, 0], parts[2][0, 0], masked)])
                return float(np.sum(out[None] * do))
            fd = np.zeros_like(q)
            for idx in np.ndindex(*q.shape):
                xp, xm = [q, k, v][i].copy(), [q, k, v][i].copy()
                xp[idx] += 1e-6
                xm[idx] -= 1e-6
                fd[idx] = (loss(xp) - loss(xm)) / 2e-6
            assert O.relative_error(got[i], fd) <= 1e-6


@pytest.mark.parametrize("masked", [True, False])
def test_f32_validation_mode_cfg1(masked):
    q, k, v, do = O.inputs(4096, 64, 1, 4, 0)
    qf, kf, vf, dof = (x.astype(np.float32).astype(np.float64) for x in (q, k, v, do))
    ref = O.lasp2_full(qf, kf, vf, dof, 2, masked)
    it = lasp2_iteration(ChunkedSequence(*(dev(x, torch.float32) for x in (q, k, v)), 2),
                         dev(do, torch.float32), masked)
    got = [to_np(cat(it.outputs))] + grads_np(it)
    for g, r in zip(got, ref):
        assert O.normalized_error(g, r) <= 1e-4


@pytest.mark.parametrize("masked", [True, False])
@pytest.mark.parametrize("n,d,h,t", [(4096, 64, 4, 2), (8192, 128, 2, 4), (3000, 128, 1, 3), (1024, 64, 2, 8)])
def test_bf16_fast_path_vs_oracle(masked, n, d, h, t):
    q, k, v, do = O.inputs(n, d, 1, h, 0)
    qb, kb, vb, dob = (O.bf16_round(x) for x in (q, k, v, do))
    ref = O.lasp2_full(qb, kb, vb, dob, t, masked)
    it = lasp2_iteration(ChunkedSequence(*(dev(x, torch.bfloat16) for x in (qb, kb, vb)), t),
                         dev(dob, torch.bfloat16), masked)
    got = [to_np(cat(it.outputs))] + grads_np(it)
    for name, g, r in zip(("out", "dq", "dk", "dv"), got, ref):
        e = O.normalized_error(g, r)
        assert e <= 1e-2, (name, e)
    assert it.run.stats.allgather_launches == 2
    assert it.run.rank_stats[0].bytes_sent == 2 * h * d * d * 4  # f32 states for bf16 data


def test_bf16_cfg1_against_reference_rows(golden):
    """The tcgen05 path on cfg1 against the reference's own (f64, unrounded) outputs."""
    rows = golden["cfg1_rows"]
    q, k, v, do = O.inputs(4096, 64, 1, 4, 0)
    it = lasp2_iteration(ChunkedSequence(*(dev(x, torch.bfloat16) for x in (q, k, v)), 2),
                         dev(do, torch.bfloat16), True)
    got = dict(zip(("out", "dq", "dk", "dv"), [to_np(cat(it.outputs))] + grads_np(it)))
    for name, arr in got.items():
        assert O.normalized_error(arr[:, :, rows], golden[f"cfg1_{name}_rows"]) <= 1e-2, name


def test_first_chunk_output_is_pure_intra():
    q, k, v, _ = O.inputs(16, 4, seed=1)
    seq = ChunkedSequence(q, k, v, 4)
    fwd = lasp2_forward_masked(seq)
    qc, kc, vc = seq.chunk(0)
    assert torch.equal(fwd.outputs[0], intra_forward(qc, kc, vc))


def test_intra_kernels_match_serial():
    q, k, v, do = O.inputs(300, 8, 2, 2, seed=7)
    out = to_np(intra_forward(q, k, v))
    g = intra_backward(q, k, v, do)
    for bi in range(2):
        for hi in range(2):
            ref = O.causal_linear_forward(q[bi, hi], k[bi, hi], v[bi, hi])
            assert np.max(np.abs(out[bi, hi] - ref)) <= 1e-10
            rq, rk, rv = O.linear_attn_serial_backward(q[bi, hi], k[bi, hi], v[bi, hi], do[bi, hi], True)
            for a, r in ((g.dq, rq), (g.dk, rk), (g.dv, rv)):
                assert O.relative_error(to_np(a)[bi, hi], r) <= 1e-12


@pytest.mark.parametrize("dtype", [torch.float64, torch.bfloat16])
def test_zero_values_and_zero_upstream(dtype):
    q, k, v, do = O.inputs(512, 64, seed=2)
    for masked in (True, False):
        it = lasp2_iteration(ChunkedSequence(dev(q, dtype), dev(k, dtype), torch.zeros_like(dev(v, dtype)), 4),
                             torch.zeros_like(dev(do, dtype)), masked)
        assert torch.count_nonzero(cat(it.outputs)) == 0
        for name in ("dq", "dk", "dv"):
            assert torch.count_nonzero(cat(getattr(g, name) for g in it.grads)) == 0


@pytest.mark.parametrize("masked", [True, False])
def test_exactly_one_launch_per_pass_and_no_p2p(masked):
    q, k, v, do = O.inputs(16, 4)
    seq = ChunkedSequence(q, k, v, 4)
    fwd = (lasp2_forward_masked if masked else lasp2_forward_nomask)(seq)
    assert fwd.run.stats.allgather_launches == 1 and fwd.run.stats.p2p_sends == 0
    bwd = (lasp2_backward_masked if masked else lasp2_backward_nomask)(seq, do, fwd.caches)
    assert bwd.run.stats.allgather_launches == 1 and bwd.run.stats.p2p_sends == 0
    it = lasp2_iteration(seq, do, masked)
    assert it.run.stats.allgather_launches == 2 and it.run.stats.communication_steps == 2


@pytest.mark.parametrize("batch,heads,d", [(1, 1, 4), (2, 4, 8)])
def test_state_bytes_independent_of_n(batch, heads, d):
    state_bytes = batch * heads * d * d * 8
    for n in (8, 32):
        q, k, v, do = O.inputs(n, d, batch, heads)
        it = lasp2_iteration(ChunkedSequence(q, k, v, 4), do, True)
        for rank in range(4):
            assert it.run.rank_stats[rank].bytes_sent == 2 * state_bytes
        assert it.run.stats.bytes_sent == 2 * 4 * state_bytes


def test_cache_contents_and_backward_validation():
    q, k, v, do = O.inputs(8, 4)
    seq = ChunkedSequence(q, k, v, 2)
    masked = lasp2_forward_masked(seq).caches
    assert all(c.masked and c.state_folds == 1 and c.m_prefix is not None and c.m_full is None for c in masked)
    nomask = lasp2_forward_nomask(seq).caches
    assert all(not c.masked and c.m_full is not None for c in nomask)
    with pytest.raises(ValueError):
        lasp2_backward_masked(seq, do, nomask)
    with pytest.raises(ValueError):
        lasp2_backward_nomask(seq, do, nomask[:1])
    qc, kc, vc = seq.chunk(0)
    hollow = [ActivationCache(q=qc, k=kc, v=vc, masked=False)] * 2
    with pytest.raises(ValueError):
        lasp2_backward_nomask(seq, do, hollow)


def test_world_shape_validation():
    q, k, v, _ = O.inputs(8, 4)
    seq = ChunkedSequence(q, k, v, 2)
    with pytest.raises(ValueError):
        lasp2_forward_masked(seq, comm.WorldConfig(world_size=4, sp_size=4))
    with pytest.raises(ValueError):
        lasp2_forward_masked(seq, comm.WorldConfig(world_size=2, element_bytes=4))


def test_overlap_schedule_agrees_and_trace_order():
    q, k, v, _ = O.inputs(1024, 64, 1, 2, seed=9)
    seq = ChunkedSequence(q, k, v, 4)
    plain = lasp2_forward_masked(seq)
    overlap = lasp2_overlap_schedule(seq)
    for a, b in zip(plain.outputs, overlap.outputs):
        # f64: both schedules add the inter term after the intra pass -> bitwise equal
        assert torch.equal(a, b)

    def kinds(run):
        order = {r: [] for r in range(4)}
        for ev in run.trace:
            if ev.kind in ("all_gather_issue", "all_gather_complete", "intra_start", "intra_end"):
                order[ev.rank].append(ev.kind)
        return order

    for ks in kinds(plain.run).values():
        assert ks == ["all_gather_issue", "all_gather_complete", "intra_start", "intra_end"]
    for ks in kinds(overlap.run).values():
        assert ks == ["all_gather_issue", "intra_start", "intra_end", "all_gather_complete"]


def test_data_parallel_replicas_share_results():
    q, k, v, do = O.inputs(8, 4, seed=11)
    seq = ChunkedSequence(q, k, v, 2)
    wide = lasp2_iteration(seq, do, True, comm.WorldConfig(world_size=4, sp_size=2))
    narrow = lasp2_iteration(seq, do, True)
    for a, b in zip(wide.outputs, narrow.outputs):
        assert torch.equal(a, b)
    assert wide.run.stats.allgather_launches == 4
    assert len(wide.run.rank_stats) == 4


def test_bf16_large_n_chunking_invariance():
    """Property at scale: the same 256K-token sequence split over T=1 and T=8
    ranks gives the same result to bf16 accuracy (N-independent exchange)."""
    from paper_2502_07563_b200.datagen import gen_slots_device
    n, d, h = 262144, 128, 2
    q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
    one = lasp2_iteration(ChunkedSequence(q, k, v, 1), do, True)
    eight = lasp2_iteration(ChunkedSequence(q, k, v, 8), do, True)
    pairs = [(one.outputs[0], cat(eight.outputs))]
    for name in ("dq", "dk", "dv"):
        pairs.append((getattr(one.grads[0], name), cat(getattr(g, name) for g in eight.grads)))
    for a, b in pairs:
        a, b = a.float(), b.float()
        assert torch.isfinite(b).all()
        assert ((a - b).abs().max() / a.abs().max()).item() <= 1e-2


def test_fused_backward_variant_matches_default():
    import paper_2502_07563_b200.lasp2 as L
    q, k, v, do = O.inputs(3000, 128, 1, 2, 0)
    seq = ChunkedSequence(*(dev(x, torch.bfloat16) for x in (q, k, v)), 3)
    a = lasp2_iteration(seq, dev(do, torch.bfloat16), True)
    L.MASKED_BWD_FUSED = True
    try:
        b = lasp2_iteration(seq, dev(do, torch.bfloat16), True)
    finally:
        L.MASKED_BWD_FUSED = False
    for name in ("dq", "dk", "dv"):
        x = cat(getattr(g, name) for g in a.grads).float()
        y = cat(getattr(g, name) for g in b.grads).float()
        assert ((x - y).abs().max() / x.abs().max()).item() <= 1e-2


@pytest.mark.parametrize("n,d,h", [(4096, 128, 16), (1000, 64, 3)])
def test_world_of_one_fused_unmasked_matches_per_step_kernels(n, d, h, monkeypatch):
    """T = 1 unmasked layer: persistent local kernels == per-step kernels (bf16) and
    the gather is still accounted once per pass (lasp2.py:208-216, :256-267)."""
    from paper_2502_07563_b200 import lasp2 as L
    q, k, v, do = O.inputs(n, d, 1, h, 9)
    q, k, v, do = (dev(x, torch.bfloat16) for x in (q, k, v, do))
    res = {}
    for mode, fused, phases in (("fused", True, True), ("phases", False, True), ("per-step", False, False)):
        monkeypatch.setattr(L, "LOCAL_FUSED", fused)
        monkeypatch.setattr(L, "FLAT_PHASES", phases)
        it = lasp2_iteration(ChunkedSequence(q, k, v, 1), do, False)
        assert it.run.stats.allgather_launches == 2
        res[mode] = [it.outputs[0]] + [getattr(it.grads[0], n_) for n_ in ("dq", "dk", "dv")]
    for a, b in zip(res["fused"], res["phases"]):  # the same kernels split around the (identity) gather
        assert torch.equal(a, b)
    for a, b in zip(res["fused"], res["per-step"]):
        scale = b.double().abs().max().item()
        assert (a.double() - b.double()).abs().max().item() <= 6e-3 * scale  # <= 1.5 bf16 ulp


@pytest.mark.parametrize("t,n,d,h", [(2, 8192, 128, 4), (4, 4000, 64, 3), (8, 2048, 128, 16)])
def test_unmasked_flat_phases_match_per_step_kernels(t, n, d, h, monkeypatch):
    """T > 1 unmasked: phase-1 / phase-2 persistent launches around the all_gather ==
    segment states + scan + apply kernels (bf16), same ledger, and against the oracle."""
    from paper_2502_07563_b200 import lasp2 as L
    q, k, v, do = O.inputs(n, d, 1, h, 21)
    xs = [dev(x, torch.bfloat16) for x in (q, k, v, do)]
    res = {}
    for phases in (True, False):
        monkeypatch.setattr(L, "FLAT_PHASES", phases)
        it = lasp2_iteration(ChunkedSequence(*xs[:3], t), xs[3], False)
        assert it.run.stats.allgather_launches == 2 and it.run.stats.p2p_sends == 0
        res[phases] = [cat(it.outputs)] + [cat(getattr(g, n_) for g in it.grads) for n_ in ("dq", "dk", "dv")]
    for a, b in zip(res[True], res[False]):
        scale = b.double().abs().max().item()
        assert (a.double() - b.double()).abs().max().item() <= 6e-3 * scale
    refs = O.lasp2_full(*(to_np(x) for x in xs), t, False)  # f64 on the same bf16-rounded inputs
    for got, ref in zip(res[True], refs):
        assert O.normalized_error(to_np(got), ref) <= 1e-2


@pytest.mark.parametrize("t", [2, 4])
def test_gathered_fused_consumer_matches_fold_then_kernel(t, monkeypatch):
    """bf16 masked, all_gather path: the chunk / dK-dV kernels folding the gathered
    states in their prologue == fold launch + seeded kernel, bit for bit (same
    copy-first order), with the same M_{1:t-1} in the cache."""
    from paper_2502_07563_b200 import lasp2 as L
    q, k, v, do = O.inputs(4096, 128, 1, 4, 31)
    xs = [dev(x, torch.bfloat16) for x in (q, k, v, do)]
    res = {}
    for fused in (True, False):
        monkeypatch.setattr(L, "GATHERED_FUSED_CONSUMER", fused)
        it = lasp2_iteration(ChunkedSequence(*xs[:3], t), xs[3], True)
        res[fused] = ([cat(it.outputs)] + [cat(getattr(g, n_) for g in it.grads) for n_ in ("dq", "dk", "dv")]
                      + [c.m_prefix for c in it.caches])
        assert it.run.stats.allgather_launches == 2
    for a, b in zip(res[True], res[False]):
        assert torch.equal(a, b)
