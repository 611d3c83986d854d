"""CPU oracle for the LASP-2 / LASP-2H hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker (never as the measured or
shipped path). It is a numpy float64 restatement of the reference algorithm
(/root/reference/pkg/src/laspsim, cited file:line per function), pinned
against outputs of the reference itself: tests/golden/make_golden.py imports
the reference in the build container and commits small fixtures that
tests/test_oracle.py checks this module against.

Differences from the reference are in grouping only:
* the reference's intra-chunk forward walks tokens one at a time
  (oracle.py:50-62) and its backward materialises C x C masks
  (lasp2.py:189-203); both are infeasible beyond C ~ 32K, so this oracle
  evaluates the same sums blockwise (Bc tokens per block, exact same terms);
* everything else (per-rank programs, ascending/descending fold order of the
  gathered states, the softmax formulas) follows the reference line by line.
"""
from __future__ import annotations

import hashlib

import numpy as np

# ---------------------------------------------------------------------------
# datagen (reference datagen.py:14-85)
# ---------------------------------------------------------------------------
_U64 = np.uint64
_GAMMA = _U64(0x9E3779B97F4A7C15)
_MIX1 = _U64(0xBF58476D1CE4E5B9)
_MIX2 = _U64(0x94D049BB133111EB)


def _mix64(z):
    """SplitMix64 finalizer, wrapping uint64 arithmetic (datagen.py:22-27)."""
    z = (z + _GAMMA) & _U64(0xFFFFFFFFFFFFFFFF)
    z = (z ^ (z >> _U64(30))) * _MIX1
    z = (z ^ (z >> _U64(27))) * _MIX2
    return z ^ (z >> _U64(31))


def _tag_word(tag: str):
    """blake2b-8 little-endian tag word (datagen.py:30-32)."""
    return _U64(int.from_bytes(hashlib.blake2b(tag.encode("utf-8"), digest_size=8).digest(), "little"))


_CGEN = []


def _c_datagen():
    """oracle/liboracle_datagen.so (oracle/datagen.c, the same formula in C with OpenMP) if built."""
    if not _CGEN:
        import ctypes
        from pathlib import Path

        lib = None
        path = Path(__file__).resolve().parent / "liboracle_datagen.so"
        if path.exists():
            try:
                lib = ctypes.CDLL(str(path))
                for nm in ("oracle_gen_data_f64", "oracle_gen_data_f32"):
                    getattr(lib, nm).argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
            except OSError:
                lib = None
        _CGEN.append(lib)
    return _CGEN[0]


def gen_data(seed: int, rows: int, cols: int, tag: str = "", dtype=np.float64) -> np.ndarray:
    """datagen.py:35-57."""
    with np.errstate(over="ignore"):
        h0 = _mix64(_U64(seed % (1 << 64)) ^ _tag_word(tag))
    lib = _c_datagen()
    dt = np.dtype(dtype)
    if lib is not None and dt in (np.dtype(np.float64), np.dtype(np.float32)) and rows * cols >= 1 << 16:
        out = np.empty((rows, cols), dtype=dt)
        fn = lib.oracle_gen_data_f64 if dt == np.float64 else lib.oracle_gen_data_f32
        fn(int(h0), rows, cols, out.ctypes.data)
        return out
    with np.errstate(over="ignore"):
        r = np.arange(rows, dtype=np.uint64)[:, None]
        c = np.arange(cols, dtype=np.uint64)[None, :]
        h = _mix64(_mix64(h0 ^ r) ^ c)
    u = (h >> _U64(11)).astype(np.float64) * 2.0 ** -53
    return (2.0 * u - 1.0).astype(dtype, copy=False)


def gen_slots(seed: int, batch: int, heads: int, rows: int, cols: int, tag: str, dtype=np.float64) -> np.ndarray:
    """datagen.py:60-71."""
    out = np.empty((batch, heads, rows, cols), dtype=dtype)
    for b in range(batch):
        for h in range(heads):
            out[b, h] = gen_data(seed, rows, cols, tag=f"{tag}/b{b}/h{h}", dtype=dtype)
    return out


def qkv_slots(seed: int, batch: int, heads: int, n: int, d: int, dtype=np.float64):
    """datagen.py:74-79."""
    return tuple(gen_slots(seed, batch, heads, n, d, t, dtype) for t in ("q", "k", "v"))


def inputs(n: int, d: int, batch: int = 1, heads: int = 1, seed: int = 0):
    """The reference tests' fixture: qkv_slots + gen_slots(..., "do") (test_lasp2.py:22-25)."""
    q, k, v = qkv_slots(seed, batch, heads, n, d)
    return q, k, v, gen_slots(seed, batch, heads, n, d, "do")


def bf16_round(x: np.ndarray) -> np.ndarray:
    """f64 -> f32 -> bf16 (round to nearest even) -> f64, as the GPU path sees its inputs."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    bits = f.view(np.uint32).astype(np.uint64)
    lsb = (bits >> np.uint64(16)) & np.uint64(1)
    bits = (bits + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return bits.astype(np.uint32).view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# numerics: ordered folds (numerics.py:71-121)
# ---------------------------------------------------------------------------

def prefix_sum_states(states, upto: int) -> np.ndarray:
    """Copy of states[0], ascending adds to upto-1; upto=0 -> zeros (numerics.py:71-90)."""
    if upto == 0:
        return np.zeros_like(states[0])
    acc = states[0].copy()
    for i in range(1, upto):
        acc += states[i]
    return acc


def suffix_sum_states(states, start: int) -> np.ndarray:
    """Copy of states[n-1], descending adds down to start; start=n -> zeros (numerics.py:93-116)."""
    n = len(states)
    if start == n:
        return np.zeros_like(states[0])
    acc = states[n - 1].copy()
    for i in range(n - 2, start - 1, -1):
        acc += states[i]
    return acc


def sum_states(states) -> np.ndarray:
    """numerics.py:119-121."""
    return prefix_sum_states(states, len(states))


# ---------------------------------------------------------------------------
# serial references (oracle.py:50-108)
# ---------------------------------------------------------------------------

def causal_linear_forward(q, k, v) -> np.ndarray:
    """Per-token recurrence o_s = q_s M_s, M_s = M_{s-1} + k_s^T v_s (oracle.py:50-62)."""
    n, d = q.shape
    m = np.zeros((d, d), dtype=q.dtype)
    out = np.empty_like(q)
    for s in range(n):
        m = m + np.outer(k[s], v[s])
        out[s] = q[s] @ m
    return out


def linear_attn_serial(q, k, v, causal: bool) -> np.ndarray:
    """oracle.py:65-74."""
    if causal:
        return causal_linear_forward(q, k, v)
    return q @ (k.T @ v)


def linear_attn_serial_backward(q, k, v, d_out, causal: bool):
    """oracle.py:77-108: (dq, dk, dv)."""
    n, d = q.shape
    if not causal:
        m = k.T @ v
        g = q.T @ d_out
        return d_out @ m.T, v @ g.T, k @ g
    states = np.empty((n, d, d))
    m = np.zeros((d, d))
    for s in range(n):
        m = m + np.outer(k[s], v[s])
        states[s] = m
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    g = np.zeros((d, d))
    for s in range(n - 1, -1, -1):
        dq[s] = d_out[s] @ states[s].T
        g += np.outer(q[s], d_out[s])
        dk[s] = v[s] @ g.T
        dv[s] = k[s] @ g
    return dq, dk, dv


# ---------------------------------------------------------------------------
# LASP-2 world restatement (lasp2.py:208-409), blocked intra terms
# ---------------------------------------------------------------------------

def _tril(n: int) -> np.ndarray:
    return np.tril(np.ones((n, n)))


def intra_forward_blocked(q, k, v, bc: int = 256) -> np.ndarray:
    """[(Q K^T) o Psi] V over one chunk, Bc-blocked (lasp2.py:168-186). Shapes (..., C, d)."""
    c = q.shape[-2]
    d = q.shape[-1]
    out = np.empty_like(q)
    s = np.zeros(q.shape[:-2] + (d, d))
    for b0 in range(0, c, bc):
        b1 = min(c, b0 + bc)
        qb, kb, vb = q[..., b0:b1, :], k[..., b0:b1, :], v[..., b0:b1, :]
        sc = (qb @ np.swapaxes(kb, -1, -2)) * _tril(b1 - b0)
        out[..., b0:b1, :] = sc @ vb + qb @ s
        s = s + np.swapaxes(kb, -1, -2) @ vb
    return out


def intra_backward_blocked(q, k, v, do, bc: int = 256):
    """Gradients of the masked intra term (lasp2.py:189-203), Bc-blocked."""
    c, d = q.shape[-2], q.shape[-1]
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    s = np.zeros(q.shape[:-2] + (d, d))
    for b0 in range(0, c, bc):  # dq with forward prefix states
        b1 = min(c, b0 + bc)
        m = _tril(b1 - b0)
        qb, kb, vb, dob = (x[..., b0:b1, :] for x in (q, k, v, do))
        ds = (dob @ np.swapaxes(vb, -1, -2)) * m
        dq[..., b0:b1, :] = ds @ kb + dob @ np.swapaxes(s, -1, -2)
        s = s + np.swapaxes(kb, -1, -2) @ vb
    g = np.zeros(q.shape[:-2] + (d, d))
    starts = list(range(0, c, bc))
    for b0 in reversed(starts):  # dk, dv with suffix states of q^T do
        b1 = min(c, b0 + bc)
        m = _tril(b1 - b0)
        qb, kb, vb, dob = (x[..., b0:b1, :] for x in (q, k, v, do))
        ds = (dob @ np.swapaxes(vb, -1, -2)) * m
        sc = (qb @ np.swapaxes(kb, -1, -2)) * m
        dk[..., b0:b1, :] = np.swapaxes(ds, -1, -2) @ qb + vb @ np.swapaxes(g, -1, -2)
        dv[..., b0:b1, :] = np.swapaxes(sc, -1, -2) @ dob + kb @ g
        g = g + np.swapaxes(qb, -1, -2) @ dob
    return dq, dk, dv


def _chunks(x: np.ndarray, t: int):
    c = x.shape[2] // t
    return [x[:, :, i * c:(i + 1) * c, :] for i in range(t)]


def lasp2_forward(q, k, v, chunks: int, masked: bool, bc: int = 256):
    """Per-rank outputs of lasp2_forward_masked/nomask (lasp2.py:208-243, 323-344).

    Returns (outputs, m_prefix or m_full per rank)."""
    qs, ks, vs = _chunks(q, chunks), _chunks(k, chunks), _chunks(v, chunks)
    states = [np.swapaxes(kc, -1, -2) @ vc for kc, vc in zip(ks, vs)]  # chunk_state, lasp2.py:130-137
    outs, reduced = [], []
    for t in range(chunks):
        if not masked:
            m_full = sum_states(states)  # lasp2.py:212
            outs.append(qs[t] @ m_full)
            reduced.append(m_full)
            continue
        out = intra_forward_blocked(qs[t], ks[t], vs[t], bc)
        m_prefix = prefix_sum_states(states, t)  # lasp2.py:236
        if t > 0:
            out = out + qs[t] @ m_prefix  # lasp2.py:238-239
        outs.append(out)
        reduced.append(m_prefix)
    return outs, reduced


def lasp2_backward(q, k, v, d_out, chunks: int, masked: bool, bc: int = 256):
    """Per-rank (dq, dk, dv) of lasp2_backward_masked/nomask (lasp2.py:256-285)."""
    qs, ks, vs, ds = (_chunks(x, chunks) for x in (q, k, v, d_out))
    states = [np.swapaxes(kc, -1, -2) @ vc for kc, vc in zip(ks, vs)]
    grads = [np.swapaxes(qc, -1, -2) @ dc for qc, dc in zip(qs, ds)]  # chunk_state_grad, lasp2.py:140-147
    out = []
    for t in range(chunks):
        if not masked:
            m_full = sum_states(states)
            dm_full = sum_states(grads)  # full sum, lasp2.py:261-263
            out.append((ds[t] @ np.swapaxes(m_full, -1, -2), vs[t] @ np.swapaxes(dm_full, -1, -2),
                        ks[t] @ dm_full))
            continue
        dq, dk, dv = intra_backward_blocked(qs[t], ks[t], vs[t], ds[t], bc)
        if t > 0:
            dq = dq + ds[t] @ np.swapaxes(prefix_sum_states(states, t), -1, -2)  # lasp2.py:278-279
        if t < chunks - 1:
            dm = suffix_sum_states(grads, t + 1)  # lasp2.py:281
            dk = dk + vs[t] @ np.swapaxes(dm, -1, -2)
            dv = dv + ks[t] @ dm
        out.append((dq, dk, dv))
    return out


def lasp2_full(q, k, v, d_out, chunks: int, masked: bool, bc: int = 256):
    """Concatenated (out, dq, dk, dv) of one lasp2_iteration (lasp2.py:390-409)."""
    outs, _ = lasp2_forward(q, k, v, chunks, masked, bc)
    grads = lasp2_backward(q, k, v, d_out, chunks, masked, bc)
    cat = lambda xs: np.concatenate(xs, axis=2)  # noqa: E731
    return cat(outs), cat([g[0] for g in grads]), cat([g[1] for g in grads]), cat([g[2] for g in grads])


def lasp1_nomask_full(q, k, v, d_out, chunks: int):
    """Concatenated (out, dq, dk, dv) of the literal exclusive-prefix ring
    (lasp1.py:43-72, 110-140): O_t = Q_t M_{1:t-1}, rank 0 zeros; the last
    chunk's k/v reach no output."""
    qs, ks, vs, ds = (_chunks(x, chunks) for x in (q, k, v, d_out))
    states = [np.swapaxes(kc, -1, -2) @ vc for kc, vc in zip(ks, vs)]
    grads = [np.swapaxes(qc, -1, -2) @ dc for qc, dc in zip(qs, ds)]
    out, dq, dk, dv = [], [], [], []
    for t in range(chunks):
        if t == 0:
            out.append(np.zeros_like(qs[t]))
            dq.append(np.zeros_like(qs[t]))
        else:
            m = prefix_sum_states(states, t)
            out.append(qs[t] @ m)
            dq.append(ds[t] @ np.swapaxes(m, -1, -2))
        if t == chunks - 1:
            dk.append(np.zeros_like(ks[t]))
            dv.append(np.zeros_like(vs[t]))
        else:
            g = suffix_sum_states(grads, t + 1)
            dk.append(vs[t] @ np.swapaxes(g, -1, -2))
            dv.append(ks[t] @ g)
    cat = lambda xs: np.concatenate(xs, axis=2)  # noqa: E731
    return cat(out), cat(dq), cat(dk), cat(dv)


# ---------------------------------------------------------------------------
# softmax / LASP-2H (oracle.py:111-158, standard_sp.py:37-76)
# ---------------------------------------------------------------------------

def softmax_probs(q, k_full, causal: bool, row_offset: int = 0) -> np.ndarray:
    """oracle.py:111-133."""
    d = q.shape[1]
    scores = (q @ k_full.T) / np.sqrt(np.asarray(d, dtype=q.dtype))
    if causal:
        rows = row_offset + np.arange(q.shape[0])[:, None]
        cols = np.arange(k_full.shape[0])[None, :]
        scores = np.where(cols <= rows, scores, -np.inf)
    scores = scores - scores.max(axis=1, keepdims=True)
    p = np.exp(scores)
    return p / p.sum(axis=1, keepdims=True)


def softmax_chunk_forward(q, k_full, v_full, causal: bool, row_offset: int = 0) -> np.ndarray:
    """oracle.py:136-139."""
    return softmax_probs(q, k_full, causal, row_offset) @ v_full


def softmax_chunk_backward(q, k_full, v_full, d_out, causal: bool, row_offset: int = 0):
    """oracle.py:142-158: (dq, dk_full, dv_full)."""
    p = softmax_probs(q, k_full, causal, row_offset)
    dv_full = p.T @ d_out
    dp = d_out @ v_full.T
    ds = p * (dp - np.sum(dp * p, axis=1, keepdims=True))
    scale = 1.0 / np.sqrt(np.asarray(q.shape[1], dtype=q.dtype))
    return (ds @ k_full) * scale, (ds.T @ q) * scale, dv_full


def cp_full(q, k, v, d_out, chunks: int, causal: bool = True):
    """Concatenated (out, dq, dk, dv) of cp_iteration (standard_sp.py:37-76, 112-127)."""
    b, h, n, d = q.shape
    c = n // chunks
    out = np.empty_like(q)
    dq = np.empty_like(q)
    contrib = []  # per rank full-length [dk; dv]
    for t in range(chunks):
        rows = slice(t * c, (t + 1) * c)
        dk_full = np.empty_like(k)
        dv_full = np.empty_like(v)
        for bi in range(b):
            for hi in range(h):
                out[bi, hi, rows] = softmax_chunk_forward(q[bi, hi, rows], k[bi, hi], v[bi, hi], causal, t * c)
                dq[bi, hi, rows], dk_full[bi, hi], dv_full[bi, hi] = softmax_chunk_backward(
                    q[bi, hi, rows], k[bi, hi], v[bi, hi], d_out[bi, hi, rows], causal, t * c)
        contrib.append(np.concatenate([dk_full, dv_full], axis=2))
    merged = sum_states(contrib)  # ascending rank fold, standard_sp.py:72
    return out, dq, merged[:, :, :n], merged[:, :, n:]


# ---------------------------------------------------------------------------
# hybrid layer stacks (hybrid.py:60-63, 136-160, 306-361)
# ---------------------------------------------------------------------------

def projection_weight(seed: int, layer: int, role: str, d: int) -> np.ndarray:
    """(d, d) weight uniform in [-1/sqrt(d), 1/sqrt(d)) (datagen.py:82-85)."""
    return gen_data(seed, d, d, tag=f"w{role}/layer{layer}") / np.sqrt(float(d))


def stack_weights(layers: str, dim: int, seed: int, round_bf16: bool = False):
    """layer_weights (hybrid.py:60-63); optionally bf16-rounded as the bf16 GPU path sees them."""
    ws = [tuple(projection_weight(seed, i, role, dim) for role in "qkv") for i in range(len(layers))]
    return [tuple(bf16_round(w) for w in t) for t in ws] if round_bf16 else ws


def stack_iteration(layers: str, x, d_out, causal: bool = True, weights=None, seed: int = 0, bc: int = 256):
    """Serial layer stack forward + analytic backward on the full sequence
    (serial_stack_oracle, hybrid.py:306-361): L layers blocked (lasp2 T=1),
    N layers per-slot softmax. Returns (out, d_x, d_weights, layer_outputs)."""
    layers = layers.replace(" ", "")
    weights = weights if weights is not None else stack_weights(layers, x.shape[-1], seed)
    retained, layer_outputs = [], []
    cur = x
    for kind, (wq, wk, wv) in zip(layers, weights):
        q, k, v = cur @ wq, cur @ wk, cur @ wv  # _project, hybrid.py:136-142
        if kind == "L":
            out = lasp2_forward(q, k, v, 1, causal, bc)[0][0]
        else:
            out = np.empty_like(q)
            for bi in range(q.shape[0]):
                for hi in range(q.shape[1]):
                    out[bi, hi] = softmax_chunk_forward(q[bi, hi], k[bi, hi], v[bi, hi], causal, 0)
        retained.append((cur, q, k, v))
        layer_outputs.append(out)
        cur = out
    dy = d_out
    d_weights = [()] * len(layers)
    for i in range(len(layers) - 1, -1, -1):
        inp, q, k, v = retained[i]
        if layers[i] == "L":
            dq, dk, dv = lasp2_backward(q, k, v, dy, 1, causal, bc)[0]
        else:
            dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
            for bi in range(q.shape[0]):
                for hi in range(q.shape[1]):
                    dq[bi, hi], dk[bi, hi], dv[bi, hi] = softmax_chunk_backward(
                        q[bi, hi], k[bi, hi], v[bi, hi], dy[bi, hi], causal, 0)
        rows = lambda a: a.reshape(-1, a.shape[-1])  # noqa: E731  pack_slots
        d_weights[i] = tuple(rows(inp).T @ rows(g) for g in (dq, dk, dv))  # _weight_grads, hybrid.py:154-160
        wq, wk, wv = weights[i]
        dy = dq @ wq.T + dk @ wk.T + dv @ wv.T  # hybrid.py:207-210
    return layer_outputs[-1], dy, d_weights, layer_outputs


# ---------------------------------------------------------------------------
# error metrics (oracle.py:230-233; SURVEY §8a note P)
# ---------------------------------------------------------------------------

def relative_error(got, ref) -> float:
    """Max entrywise |got - ref| / max(1, |ref|) (oracle.py:230-233)."""
    denom = np.maximum(1.0, np.abs(ref))
    return float(np.max(np.abs(np.asarray(got, dtype=np.float64) - ref) / denom))


def normalized_error(got, ref) -> float:
    """max|got - ref| / max|ref| — the parity metric for bf16 / fp32 modes (SURVEY §8a note P)."""
    ref = np.asarray(ref, dtype=np.float64)
    scale = float(np.max(np.abs(ref)))
    err = float(np.max(np.abs(np.asarray(got, dtype=np.float64) - ref)))
    return err / scale if scale > 0 else err
