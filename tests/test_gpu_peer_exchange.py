"""Fused peer-memory state exchange: the scan kernel stores the
chunk total into every rank's receive buffer and releases epoch-stamped flags;
the fold waits on the flags it needs. On one GPU the ranks are host threads
(buffers on the same device), which exercises the kernels, the flag protocol
and the drivers; over NVLink the same kernels get symmetric-memory peer
addresses. Results must equal the all_gather path bit for bit (same scan, same
fold) and match the oracle."""
import numpy as np
import pytest
import torch

from oracle import lasp_oracle as O
from paper_2502_07563_b200 import comm, lasp2, ops
from paper_2502_07563_b200._lib import FOLD_FULL, FOLD_PREFIX, FOLD_SUFFIX
from paper_2502_07563_b200.lasp2 import ChunkedSequence, lasp2_iteration

pytestmark = pytest.mark.gpu


@pytest.fixture
def peer_mode():
    old = lasp2.STATE_EXCHANGE
    lasp2.STATE_EXCHANGE = "peer"
    yield
    lasp2.STATE_EXCHANGE = old


def cat(xs):
    return torch.cat(list(xs), dim=2).double().cpu().numpy()


def grads(it):
    return [cat(getattr(g, nm) for g in it.grads) for nm in ("dq", "dk", "dv")]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("t", [1, 2, 5])
def test_scan_put_and_fold_equal_gather(dtype, t):
    """Kernel level, one stream: every rank puts, then every rank folds."""
    b, h, nseg, d = 1, 3, 4, 16
    dev = torch.device("cuda")
    segs = [torch.randn((b, h, nseg, d, d), dtype=dtype, device=dev) for _ in range(t)]
    recv = [torch.zeros((2, t, b, h, d, d), dtype=dtype, device=dev) for _ in range(t)]
    flags = [torch.zeros(t, dtype=torch.int64, device=dev) for _ in range(t)]
    acks = [torch.zeros(t, dtype=torch.int64, device=dev) for _ in range(t)]
    done = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(t)]
    tables = [comm._ptr_table(x, dev) for x in (recv, flags, acks)]
    exs = [comm.PeerExchange(r, t, recv[r], flags[r], acks[r], done[r], *tables) for r in range(t)]
    for rnd in range(3):  # epochs advance; buffers and counters are reused
        seg_ref = [s.clone() for s in segs]
        totals = [ops.scan_segments(s, False, dtype) for s in seg_ref]
        seg_put = [s.clone() for s in segs]
        mine = [ops.scan_put(s, False, dtype, ex) for s, ex in zip(seg_put, exs)]
        gathered = torch.stack(totals)
        for r in range(t):
            assert torch.equal(mine[r], totals[r]) and torch.equal(seg_put[r], seg_ref[r])
            assert torch.equal(ops.exchange_fold(exs[r], FOLD_PREFIX, r), ops.fold(gathered, FOLD_PREFIX, r))
            assert torch.equal(ops.exchange_fold(exs[r], FOLD_SUFFIX, r + 1), ops.fold(gathered, FOLD_SUFFIX, r + 1))
            assert torch.equal(ops.exchange_fold(exs[r], FOLD_FULL), ops.fold(gathered, FOLD_FULL))
            assert flags[r].tolist() == [rnd + 1] * t and done[r].item() == 0
        for r in range(t):
            assert acks[r].tolist() == [rnd + 1] * t  # every reader acknowledged this epoch
        segs = [s * 0.5 + 1.0 for s in segs]


@pytest.mark.parametrize("masked", [True, False])
@pytest.mark.parametrize("t", [2, 4])
def test_f64_iteration_matches_reference(golden, peer_mode, masked, t):
    n, d, b, h, seed = (256, 4, 1, 1, 0) if t == 2 else (64, 16, 1, 1, 0)  # reference_cases.npz grid
    q, k, v, do = O.inputs(n, d, b, h, seed)
    key = f"lasp2_{'m' if masked else 'u'}_{n}_{d}_{t}_{b}_{h}_{seed}"
    it = lasp2_iteration(ChunkedSequence(q, k, v, t), do, masked)
    assert np.max(np.abs(cat(it.outputs) - golden[key + "_out"])) <= 1e-10
    for got, nm in zip(grads(it), ("dq", "dk", "dv")):
        assert O.relative_error(got, golden[f"{key}_{nm}"]) <= 1e-12, nm
    st = it.run.stats
    assert st.allgather_launches == 2 and st.communication_steps == 2
    assert all("peer" in ev.detail for ev in it.run.trace if ev.kind == "all_gather_issue")


@pytest.mark.parametrize("masked,overlap", [(True, False), (True, True), (False, False)])
def test_bf16_peer_equals_collective_bitwise(masked, overlap):
    n, d, b, h, t = 8192, 128, 1, 2, 4
    q, k, v, do = (torch.from_numpy(O.bf16_round(x)).to("cuda", torch.bfloat16) for x in O.inputs(n, d, b, h, 3))
    seq = ChunkedSequence(q, k, v, t)
    old = lasp2.STATE_EXCHANGE
    try:
        lasp2.STATE_EXCHANGE = "collective"
        ref = lasp2_iteration(seq, do, masked, overlap=overlap)
        lasp2.STATE_EXCHANGE = "peer"
        got = lasp2_iteration(seq, do, masked, overlap=overlap)
    finally:
        lasp2.STATE_EXCHANGE = old
    assert np.array_equal(cat(got.outputs), cat(ref.outputs))
    for a, bb in zip(grads(got), grads(ref)):
        assert np.array_equal(a, bb)
    assert got.run.stats.allgather_launches == ref.run.stats.allgather_launches == 2
    assert got.run.stats.bytes_sent == ref.run.stats.bytes_sent


def test_repeated_iterations_in_one_world(peer_mode):
    """Epochs advance across exchanges of the same buffers inside one world."""
    n, d, b, h, t = 1024, 64, 1, 2, 2
    q, k, v, do = (torch.from_numpy(O.bf16_round(x)).to("cuda", torch.bfloat16) for x in O.inputs(n, d, b, h, 4))
    seq = ChunkedSequence(q, k, v, t)
    d_chunks = lasp2._split_like(seq, do)

    def program(ctx, qc, kc, vc, dc):
        res = []
        for _ in range(3):
            out, cache = lasp2.rank_forward(ctx, qc, kc, vc, masked=True)
            g = lasp2.rank_backward(ctx, cache, dc)
            res.append((out, g.dq, g.dk, g.dv))
        return res

    run = lasp2._spawn(seq, None, program, extra_args=[(d_chunks[r],) for r in range(t)])
    for r in range(t):
        first = run.results[r][0]
        for later in run.results[r][1:]:
            assert all(torch.equal(a, bb) for a, bb in zip(first, later))
    assert run.stats.allgather_launches == 6


def test_forward_only_loop_with_a_rank_running_ahead(peer_mode):
    """Masked forward only: rank 0 needs no peer state, so nothing but the ack
    back-pressure keeps it from overwriting slots the others have not folded.
    Rank 0 runs 6 forwards before the others start (host-side delay); every
    rank's outputs must still match its first forward."""
    import threading
    n, d, b, h, t = 3072, 128, 1, 2, 3
    q, k, v, _ = (torch.from_numpy(O.bf16_round(x)).to("cuda", torch.bfloat16) for x in O.inputs(n, d, b, h, 6))
    seq = ChunkedSequence(q, k, v, t)
    gate = threading.Event()

    def program(ctx, qc, kc, vc):
        if ctx.sp_position != 0:
            gate.wait(timeout=30)
        outs = []
        for i in range(6):
            k_i = kc * (1.0 + 0.5 * i)  # a different state every epoch
            out, _ = lasp2.rank_forward(ctx, qc, k_i.contiguous(), vc, masked=True)
            outs.append(out)
            if ctx.sp_position == 0 and i == 5:
                gate.set()
        return outs

    run = lasp2._spawn(seq, None, program)
    ref = lasp2.STATE_EXCHANGE
    try:
        lasp2.STATE_EXCHANGE = "collective"
        want = lasp2._spawn(seq, None, program)
    finally:
        lasp2.STATE_EXCHANGE = ref
    for r in range(t):
        for a, bb in zip(run.results[r], want.results[r]):
            assert torch.equal(a, bb)


def test_fused_consumers_equal_wait_fold_then_kernel():
    """lasp2_causal_chunk_x / lasp2_dkdv_chunk_x (in-kernel flag wait + fold of the
    exchanged states) against exchange_fold + the plain kernels, bit for bit. All
    puts are issued first on one stream, so no consumer can spin on a producer
    that has no SM left (the drivers use the fused consumers only with one GPU per rank)."""
    t_world, n, d, h = 3, 2048, 128, 2
    dev = torch.device("cuda")
    g = torch.Generator(device="cuda").manual_seed(11)
    mk = lambda: ((torch.rand((1, h, n, d), generator=g, device=dev) * 2 - 1)).to(torch.bfloat16)  # noqa: E731
    data = [tuple(mk() for _ in range(4)) for _ in range(t_world)]  # q, k, v, do per rank
    nseg = ops.num_segments(data[0][0])

    def exchange(tag_dtype=torch.float32):
        recv = [torch.zeros((2, t_world, 1, h, d, d), dtype=tag_dtype, device=dev) for _ in range(t_world)]
        flags = [torch.zeros(t_world, dtype=torch.int64, device=dev) for _ in range(t_world)]
        acks = [torch.zeros(t_world, dtype=torch.int64, device=dev) for _ in range(t_world)]
        done = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(t_world)]
        tables = [comm._ptr_table(x, dev) for x in (recv, flags, acks)]
        return [comm.PeerExchange(r, t_world, recv[r], flags[r], acks[r], done[r], *tables) for r in range(t_world)]

    ex_f, ex_b = exchange(), exchange()
    segs = [ops.segment_states(k, v, nseg) for (_, k, v, _) in data]
    totals = [ops.scan_put(s, False, torch.bfloat16, e) for s, e in zip(segs, ex_f)]
    gsegs = [ops.segment_states(q, do, nseg) for (q, _, _, do) in data]
    gtot = [ops.scan_put(s, True, torch.bfloat16, e) for s, e in zip(gsegs, ex_b)]
    gathered, ggathered = torch.stack(totals), torch.stack(gtot)
    for r, (q, k, v, do) in enumerate(data):
        base_out = torch.empty((1, h, d, d), dtype=torch.float32, device=dev)
        got = ops.causal_chunk_x(q, k, v, segs[r], ex_f[r], r, nseg, base_out=base_out)
        m_prefix = ops.fold(gathered, FOLD_PREFIX, r)
        want = ops.causal_chunk(q, k, v, segs[r], m_prefix if r > 0 else None, nseg)
        assert torch.equal(got, want) and torch.equal(base_out, m_prefix), r
        dk, dv = ops.dkdv_chunk_x(q, k, v, do, gsegs[r], ex_b[r], r + 1, nseg)
        rr = ops.fold(ggathered, FOLD_SUFFIX, r + 1)
        wk, wv = ops.dkdv_chunk(q, k, v, do, gsegs[r], rr if r < t_world - 1 else None, nseg)
        assert torch.equal(dk, wk) and torch.equal(dv, wv), r
    torch.cuda.synchronize()
    for e in ex_f + ex_b:
        assert e.acks.tolist() == [1] * t_world  # every consumer acknowledged the epoch
