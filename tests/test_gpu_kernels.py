"""Kernel-level parity of every C-ABI entry point against fp64 torch math on the
same (bf16-rounded where applicable) inputs. Runs on a B200 only."""
import numpy as np
import pytest
import torch

from paper_2502_07563_b200 import _lib, datagen, ops

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2   # north star: bf16-in / fp32-accumulate, normalised max error
F32_TOL = 1e-4    # north star: fp32 validation mode
F64_TOL = 1e-12


def nerr(got: torch.Tensor, ref: torch.Tensor) -> float:
    got, ref = got.double(), ref.double()
    scale = ref.abs().max().item()
    e = (got - ref).abs().max().item()
    return e / scale if scale > 0 else e


def seg_ranges(nseg: int, tokens: int):
    nblk = (tokens + 127) // 128
    for s in range(nseg):
        lo, hi = (s * nblk // nseg) * 128, ((s + 1) * nblk // nseg) * 128
        yield min(lo, tokens), min(hi, tokens)


def rand(shape, dtype, seed=0, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return ((torch.rand(shape, generator=g, device="cuda", dtype=torch.float64) * 2 - 1) * scale).to(dtype)


def ref_segment_states(x, y, nseg):
    b, h, n, d = x.shape
    out = []
    for lo, hi in seg_ranges(nseg, n):
        xs, ys = x[:, :, lo:hi].double(), y[:, :, lo:hi].double()
        out.append(xs.transpose(-1, -2) @ ys)
    return torch.stack(out, dim=2)


def ref_causal(q, k, v, seg, base, nseg, reverse, transpose):
    b, h, n, d = q.shape
    out = torch.empty((b, h, n, d), dtype=torch.float64, device=q.device)
    for g, (lo, hi) in enumerate(seg_ranges(nseg, n)):
        s0 = torch.zeros((b, h, d, d), dtype=torch.float64, device=q.device)
        if seg is not None:
            s0 = s0 + seg[:, :, g].double()
        if base is not None:
            s0 = s0 + base.double()
        if transpose:
            s0 = s0.transpose(-1, -2)
        qs, ks, vs = (x[:, :, lo:hi].double() for x in (q, k, v))
        L = hi - lo
        m = torch.ones((L, L), dtype=torch.float64, device=q.device)
        m = torch.triu(m) if reverse else torch.tril(m)
        out[:, :, lo:hi] = ((qs @ ks.transpose(-1, -2)) * m) @ vs + qs @ s0
    return out


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (2, 1)])
def test_probe_gemm_descriptor_conventions(a_mn, b_mn):
    """a_mn 2: A staged into TMEM (bf16 pairs along K) and read by the TS-mode MMA."""
    a = rand((128, 128), torch.bfloat16, 1)
    b = rand((128, 128), torch.bfloat16, 2)
    d = ops.probe_gemm(a, b, a_mn, bool(b_mn))
    A = a.double().T if a_mn == 1 else a.double()  # op(A): [M][K]
    B = b.double().T if b_mn else b.double()  # op(B): [N][K]
    ref = A @ B.T
    torch.cuda.synchronize()
    assert nerr(d, ref) <= 1e-5


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("shape", [(1, 2, 1024, 128), (2, 1, 700, 64), (1, 3, 128, 32), (1, 1, 5, 8)])
def test_segment_states_and_scan(dtype, shape):
    x, y = rand(shape, dtype, 3), rand(shape, dtype, 4)
    nseg = max(1, min(3, (shape[2] + 127) // 128))
    seg = ops.segment_states(x, y, nseg)
    ref = ref_segment_states(x, y, nseg)
    tol = {torch.bfloat16: 1e-5, torch.float32: 1e-5, torch.float64: F64_TOL}[dtype]
    assert nerr(seg, ref) <= tol
    fwd = seg.clone()
    total = ops.scan_segments(fwd, reverse=False, data_dtype=dtype)
    assert nerr(total, ref.sum(2)) <= tol
    assert torch.count_nonzero(fwd[:, :, 0]) == 0
    for g in range(1, nseg):
        assert nerr(fwd[:, :, g], ref[:, :, :g].sum(2)) <= tol
    rev = seg.clone()
    ops.scan_segments(rev, reverse=True, data_dtype=dtype)
    assert torch.count_nonzero(rev[:, :, nseg - 1]) == 0
    for g in range(nseg - 1):
        assert nerr(rev[:, :, g], ref[:, :, g + 1:].sum(2)) <= tol


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("reverse,transpose", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("shape,nseg", [((1, 2, 1024, 128), 3), ((2, 1, 1000, 64), 2), ((1, 2, 256, 128), 1),
                                        ((1, 1, 77, 128), 1)])
def test_causal_chunk(dtype, reverse, transpose, shape, nseg):
    q, k, v = rand(shape, dtype, 5), rand(shape, dtype, 6), rand(shape, dtype, 7)
    b, h, n, d = shape
    sd = _lib.state_dtype(dtype)
    seg = rand((b, h, nseg, d, d), sd, 8, scale=30.0)
    base = rand((b, h, d, d), sd, 9, scale=30.0)
    got = ops.causal_chunk(q, k, v, seg, base, nseg, reverse=reverse, transpose_state=transpose)
    ref = ref_causal(q, k, v, seg, base, nseg, reverse, transpose)
    tol = {torch.bfloat16: BF16_TOL, torch.float32: F32_TOL, torch.float64: F64_TOL}[dtype]
    e = nerr(got, ref)
    assert e <= tol, e
    if dtype == torch.bfloat16:
        assert e <= 5e-3, e  # bf16 output rounding + bf16 state operand


def test_causal_chunk_without_states():
    q, k, v = (rand((1, 2, 512, 128), torch.bfloat16, s) for s in (10, 11, 12))
    got = ops.causal_chunk(q, k, v, None, None, 1)
    assert nerr(got, ref_causal(q, k, v, None, None, 1, False, False)) <= 5e-3


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("shape", [(1, 2, 4096, 128), (2, 2, 300, 64), (1, 1, 3, 16), (1, 2, 65536 + 77, 128)])
def test_apply_state(dtype, transpose, shape):
    x = rand(shape, dtype, 13)
    b, h, n, d = shape
    m = rand((b, h, d, d), _lib.state_dtype(dtype), 14, scale=10.0)
    got = ops.apply_state(x, m, transpose=transpose)
    mm = m.double().transpose(-1, -2) if transpose else m.double()
    ref = x.double() @ mm
    tol = {torch.bfloat16: 5e-3, torch.float32: F32_TOL, torch.float64: F64_TOL}[dtype]
    assert nerr(got, ref) <= tol
    acc = got.clone()
    ops.apply_state(x, m, transpose=transpose, out=acc, accumulate=True)
    assert nerr(acc, 2 * ref) <= tol


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fold_states_order_and_empty(dtype):
    g = rand((4, 3, 5), dtype, 15)
    g[:, 0, 0] = -0.0
    atol = 1e-12 if dtype == torch.float64 else 1e-6
    for upto in range(5):
        got = ops.prefix_states(g, upto)
        want = torch.zeros_like(g[0]) if upto == 0 else g[:upto].sum(0)
        assert torch.allclose(got, want, atol=atol, rtol=0)
    assert torch.signbit(ops.prefix_states(g, 2)[0, 0])  # copy-first keeps -0.0
    for start in range(5):
        got = ops.suffix_states(g, start)
        want = torch.zeros_like(g[0]) if start == 4 else g[start:].sum(0)
        assert torch.allclose(got, want, atol=atol, rtol=0)
    # descending fold order for suffix, ascending for prefix: exact f64 recomputation
    acc = g[3].clone()
    for i in (2, 1):
        acc += g[i]
    assert torch.equal(ops.suffix_states(g, 1), acc)
    assert torch.equal(ops.sum_states(g), ((g[0] + g[1]) + g[2]) + g[3])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
def test_gen_slots_device_bit_exact(dtype):
    got = datagen.gen_slots_device(0, 2, 3, 257, 64, "q", dtype=dtype)
    host = datagen.gen_slots(0, 2, 3, 257, 64, "q", dtype=np.float64)
    want = torch.from_numpy(host).cuda()
    if dtype == torch.float64:
        assert torch.equal(got, want)
    else:
        assert torch.equal(got, want.float().to(dtype))


def test_ops_reject_cpu_and_noncontiguous():
    x = torch.zeros((1, 1, 128, 128), dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="CUDA"):
        ops.segment_states(x, x, 1)
    y = torch.zeros((1, 1, 128, 256), dtype=torch.bfloat16, device="cuda")[..., ::2]
    with pytest.raises(ValueError, match="contiguous"):
        ops.apply_state(y, torch.zeros((1, 1, 128, 128), device="cuda"))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("shape,nseg", [((1, 2, 1024, 128), 3), ((2, 1, 1000, 64), 2), ((1, 3, 2048, 128), 9),
                                        ((1, 1, 77, 128), 1)])
def test_dkdv_pair_matches_two_passes(dtype, shape, nseg):
    q, k, v, do = (rand(shape, dtype, s) for s in (21, 22, 23, 24))
    b, h, n, d = shape
    sd = _lib.state_dtype(dtype)
    seg = rand((b, h, nseg, d, d), sd, 25, scale=30.0)
    base = rand((b, h, d, d), sd, 26, scale=30.0)
    dk, dv = ops.dkdv_chunk(q, k, v, do, seg, base, nseg)
    rk = ref_causal(v, do, q, seg, base, nseg, True, True)
    rv = ref_causal(k, q, do, seg, base, nseg, True, False)
    tol = {torch.bfloat16: 5e-3, torch.float32: F32_TOL, torch.float64: F64_TOL}[dtype]
    assert nerr(dk, rk) <= tol
    assert nerr(dv, rv) <= tol


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("shape,nseg", [((1, 2, 1024, 128), 3), ((2, 1, 1000, 64), 2), ((1, 3, 2048, 128), 9),
                                        ((1, 1, 77, 128), 1), ((1, 2, 300, 32), 2)])
def test_dq_chunk_matches_separate_passes(dtype, shape, nseg):
    """lasp2_dq_chunk = causal_chunk(dO, V, K; S^T) and segment_states(Q, dO) in one pass."""
    q, k, v, do = (rand(shape, dtype, s) for s in (41, 42, 43, 44))
    b, h, n, d = shape
    sd = _lib.state_dtype(dtype)
    seg = rand((b, h, nseg, d, d), sd, 45, scale=30.0)
    base = rand((b, h, d, d), sd, 46, scale=30.0)
    for bs in (base, None):
        dq, gseg = ops.dq_chunk(q, k, v, do, seg, bs, nseg)
        rq = ref_causal(do, v, k, seg, bs, nseg, False, True)
        tol = {torch.bfloat16: 5e-3, torch.float32: F32_TOL, torch.float64: F64_TOL}[dtype]
        tol_s = {torch.bfloat16: 1e-5, torch.float32: 1e-5, torch.float64: F64_TOL}[dtype]
        assert nerr(dq, rq) <= tol
        assert nerr(gseg, ref_segment_states(q, do, nseg)) <= tol_s
    if dtype == torch.bfloat16:  # bitwise the same dQ as the standalone causal pass
        dq2 = ops.causal_chunk(do, v, k, seg, base, nseg, reverse=False, transpose_state=True)
        dq, _ = ops.dq_chunk(q, k, v, do, seg, base, nseg)
        assert torch.equal(dq, dq2)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("shape", [(1, 2, 4096, 128), (2, 1, 700, 64), (1, 3, 300, 32)])
def test_state_apply_and_apply2(dtype, shape):
    q, do, v, k = (rand(shape, dtype, s) for s in (31, 32, 33, 34))
    b, h, n, d = shape
    nseg = max(1, min(3, (n + 127) // 128))
    m = rand((b, h, d, d), _lib.state_dtype(dtype), 35, scale=10.0)
    seg, dq = ops.state_apply(q, do, m, nseg)
    tol_s = {torch.bfloat16: 1e-5, torch.float32: 1e-5, torch.float64: F64_TOL}[dtype]
    tol_o = {torch.bfloat16: 5e-3, torch.float32: F32_TOL, torch.float64: F64_TOL}[dtype]
    assert nerr(seg, ref_segment_states(q, do, nseg)) <= tol_s
    assert nerr(dq, do.double() @ m.double().transpose(-1, -2)) <= tol_o
    dk, dv = ops.apply_state2(v, k, m)
    assert nerr(dk, v.double() @ m.double().transpose(-1, -2)) <= tol_o
    assert nerr(dv, k.double() @ m.double()) <= tol_o


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("shape,nseg", [((1, 2, 1024, 128), 3), ((2, 1, 1000, 64), 2), ((1, 3, 2048, 128), 9),
                                        ((1, 1, 77, 128), 1)])
def test_backward_chunk_matches_separate_passes(dtype, shape, nseg):
    q, k, v, do = (rand(shape, dtype, s) for s in (41, 42, 43, 44))
    b, h, n, d = shape
    sd = _lib.state_dtype(dtype)
    # forward states: exclusive prefixes of K^T V per segment + chunk total, as the forward scan leaves them
    fseg = ops.segment_states(k, v, nseg)
    ftot = ops.scan_segments(fseg, reverse=False, data_dtype=dtype)
    fbase = rand((b, h, d, d), sd, 45, scale=30.0)
    gseg = rand((b, h, nseg, d, d), sd, 46, scale=30.0)
    gbase = rand((b, h, d, d), sd, 47, scale=30.0)
    dq, dk, dv = ops.backward_chunk(q, k, v, do, fseg, ftot, fbase, gseg, gbase, nseg)
    rq = ref_causal(do, v, k, fseg, fbase, nseg, False, True)
    rk = ref_causal(v, do, q, gseg, gbase, nseg, True, True)
    rv = ref_causal(k, q, do, gseg, gbase, nseg, True, False)
    tol = {torch.bfloat16: 6e-3, torch.float32: F32_TOL, torch.float64: F64_TOL}[dtype]
    assert nerr(dq, rq) <= tol
    assert nerr(dk, rk) <= tol
    assert nerr(dv, rv) <= tol


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("shape,nseg", [((1, 2, 1024, 128), 3), ((2, 1, 1000, 64), 2), ((1, 3, 2048, 128), 9),
                                        ((1, 1, 77, 128), 1)])
def test_backward_chunk_fwd_matches_separate_passes(dtype, shape, nseg):
    """Forward-walking single-launch backward: dK / dV from the suffix inclusive of each
    block (seeded from the neighbouring segment's exclusive scan or the chunk total)."""
    q, k, v, do = (rand(shape, dtype, s) for s in (51, 52, 53, 54))
    b, h, n, d = shape
    sd = _lib.state_dtype(dtype)
    fseg = ops.segment_states(k, v, nseg)
    ops.scan_segments(fseg, reverse=False, data_dtype=dtype)
    fbase = rand((b, h, d, d), sd, 55, scale=30.0)
    gseg = ops.segment_states(q, do, nseg)
    gtot = ops.scan_segments(gseg, reverse=True, data_dtype=dtype)  # exclusive suffix scan + chunk total
    gbase = rand((b, h, d, d), sd, 57, scale=30.0)
    dq, dk, dv = ops.backward_chunk_fwd(q, k, v, do, fseg, fbase, gseg, gtot, gbase, nseg)
    rq = ref_causal(do, v, k, fseg, fbase, nseg, False, True)
    rk = ref_causal(v, do, q, gseg, gbase, nseg, True, True)
    rv = ref_causal(k, q, do, gseg, gbase, nseg, True, False)
    tol = {torch.bfloat16: 6e-3, torch.float32: F32_TOL, torch.float64: F64_TOL}[dtype]
    assert nerr(dq, rq) <= tol
    assert nerr(dk, rk) <= tol
    assert nerr(dv, rv) <= tol


def ref_nomask_local(q, k, v, do, m_in):
    qd, kd, vd, dod = (x.double() for x in (q, k, v, do))
    m = kd.transpose(-1, -2) @ vd
    dm = qd.transpose(-1, -2) @ dod
    mi = m_in.double()
    return m, qd @ m, dod @ mi.transpose(-1, -2), vd @ dm.transpose(-1, -2), kd @ dm


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("shape", [(1, 16, 4096, 128), (2, 3, 1000, 64), (1, 2, 256, 128), (1, 1, 77, 128),
                                   (3, 50, 128, 32), (1, 16, 16384, 128)])
def test_nomask_local_forward_backward(dtype, shape):
    """World-of-one persistent kernels: flat (slot, block) split over all SMs, pieces
    crossing slot boundaries, ragged last blocks, fewer blocks than SMs."""
    if dtype != torch.bfloat16 and shape[2] > 4096:
        pytest.skip("validation kernels: small shapes only")
    q, k, v, do = (rand(shape, dtype, s) for s in (51, 52, 53, 54))
    out, m = ops.nomask_forward_local(q, k, v)
    dq, dk, dv = ops.nomask_backward_local(q, k, v, do, m)
    rm, ro, rdq, rdk, rdv = ref_nomask_local(q, k, v, do, m)
    tol_s = {torch.bfloat16: 1e-5, torch.float32: 1e-5, torch.float64: F64_TOL}[dtype]
    tol_o = {torch.bfloat16: 6e-3, torch.float32: F32_TOL, torch.float64: F64_TOL}[dtype]
    assert nerr(m, rm) <= tol_s
    for got, ref in ((out, ro), (dq, rdq), (dk, rdk), (dv, rdv)):
        assert nerr(got, ref) <= tol_o


def test_nomask_local_deterministic_and_barrier_reuse():
    """Repeated calls with different grid sizes reuse the zeroed barrier words and
    give bitwise identical results (ordered reduction, no float atomics)."""
    shapes = [(1, 16, 4096, 128), (1, 2, 256, 128), (1, 16, 4096, 128), (2, 3, 1000, 64)]
    first = {}
    for rep in range(3):
        for shape in shapes:
            q, k, v, do = (rand(shape, torch.bfloat16, s) for s in (61, 62, 63, 64))
            out, m = ops.nomask_forward_local(q, k, v)
            grads = ops.nomask_backward_local(q, k, v, do, m)
            res = [out, m, *grads]
            if shape in first:
                for a, b in zip(first[shape], res):
                    assert torch.equal(a, b)
            else:
                first[shape] = res
    ws = ops.local_workspace(torch.empty(1, 16, 4096, 128, dtype=torch.bfloat16, device="cuda"))
    torch.cuda.synchronize()
    assert int(ws[:8].view(torch.int32)[0]) == 0  # arrival counter back at zero


def test_nomask_local_workspace_validation():
    x = rand((1, 2, 256, 128), torch.bfloat16, 1)
    m = torch.empty(1, 2, 128, 128, dtype=torch.float32, device="cuda")
    small = torch.zeros(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="workspace too small"):
        ops.call("lasp2_nomask_forward_local", _lib.BF16, ops.ptr(x), ops.ptr(x), ops.ptr(x), ops.ptr(x),
                 ops.ptr(m), ops.ptr(small), small.numel(), 2, 256, 128, ops.stream_ptr())


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("shape", [(1, 4, 640, 128), (2, 2, 300, 64)])
def test_project_shared_weights(dtype, shape):
    """lasp2_project (hybrid.py:136-151): X W and X W^T with one weight for every slot, the
    accumulate form, and the three-term chain-rule sum dQ W_Q^T + dK W_K^T + dV W_V^T
    (one accumulator) against an f64 torch reference of the same rounded operands."""
    d = shape[-1]
    sd = torch.float64 if dtype == torch.float64 else torch.float32
    xs = [rand(shape, dtype, 70 + i) for i in range(3)]
    ws = [rand((d, d), dtype, 80 + i).to(sd) for i in range(3)]  # weights rounded to the data dtype
    tol = {torch.bfloat16: 1e-2, torch.float32: 1e-5, torch.float64: 1e-12}[dtype]

    def ref(terms):
        return sum(x.double() @ w.double() for x, w in terms)

    def err(got, want):
        return ((got.double() - want).abs().max() / want.abs().max()).item()

    assert err(ops.project([xs[0]], [ws[0]]), ref([(xs[0], ws[0])])) <= tol
    assert err(ops.project([xs[0]], [ws[0]], transpose=True), ref([(xs[0], ws[0].t())])) <= tol
    out = ops.project([xs[0]], [ws[0]])
    ops.project([xs[1]], [ws[1]], out=out, accumulate=True)
    assert err(out, ref([(xs[0], ws[0]), (xs[1], ws[1])])) <= 2 * tol
    three = ops.project(xs, ws, transpose=True)
    assert err(three, ref([(x, w.t()) for x, w in zip(xs, ws)])) <= tol
    with pytest.raises(ValueError):
        ops.project(xs[:2], ws[:2])
