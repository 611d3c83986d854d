"""Typed torch-facing wrappers over the C-ABI kernels.

Every function takes contiguous CUDA tensors in the BHND layout
((B, H, tokens, d) data, (B, H, d, d) states), enqueues on the current CUDA
stream and returns new tensors; the library itself never allocates.
"""
from __future__ import annotations

import ctypes
from collections import OrderedDict

import torch

from . import _lib
from ._lib import FOLD_FULL, FOLD_PREFIX, FOLD_SUFFIX, call, dtype_code, ptr, require_cuda, state_dtype, stream_ptr

_SM_COUNT: dict[int, int] = {}


def sm_count(device: torch.device | None = None) -> int:
    dev = torch.cuda.current_device() if device is None else device.index
    if dev not in _SM_COUNT:
        _SM_COUNT[dev] = torch.cuda.get_device_properties(dev).multi_processor_count
    return _SM_COUNT[dev]


def _slots(x: torch.Tensor) -> tuple[int, int, int]:
    if x.ndim != 4:
        raise ValueError(f"expected (batch, heads, tokens, dim), got {tuple(x.shape)}")
    b, h, n, d = x.shape
    return b * h, n, d


def num_segments(x: torch.Tensor) -> int:
    slots, n, d = _slots(x)
    return int(_lib.load().lasp2_num_segments(dtype_code(x.dtype), slots, n, d, sm_count(x.device)))


def segment_states(x: torch.Tensor, y: torch.Tensor, nseg: int) -> torch.Tensor:
    """(B,H,nseg,d,d): per-segment X^T Y (lasp2.py:130-147 per segment)."""
    require_cuda(x, y)
    if x.shape != y.shape or x.dtype != y.dtype:
        raise ValueError(f"segment_states operands differ: {tuple(x.shape)} {tuple(y.shape)}")
    slots, n, d = _slots(x)
    b, h = x.shape[:2]
    out = torch.empty((b, h, nseg, d, d), dtype=state_dtype(x.dtype), device=x.device)
    call("lasp2_segment_states", dtype_code(x.dtype), ptr(x), ptr(y), ptr(out), slots, n, d, nseg, stream_ptr())
    return out


def scan_segments(seg: torch.Tensor, reverse: bool, data_dtype: torch.dtype) -> torch.Tensor:
    """In place exclusive prefix (suffix if reverse) over segments; returns the chunk total (B,H,d,d)."""
    require_cuda(seg)
    b, h, nseg, d, _ = seg.shape
    total = torch.empty((b, h, d, d), dtype=seg.dtype, device=seg.device)
    call("lasp2_scan_segments", dtype_code(data_dtype), ptr(seg), ptr(total), b * h, nseg, d, int(reverse),
         stream_ptr())
    return total


def chunk_states(x: torch.Tensor, y: torch.Tensor, reverse: bool = False) -> tuple[torch.Tensor, torch.Tensor, int]:
    """Segment states scanned in place plus the chunk total (the rank's M_t)."""
    nseg = num_segments(x)
    seg = segment_states(x, y, nseg)
    total = scan_segments(seg, reverse, x.dtype)
    return seg, total, nseg


def scan_put(seg: torch.Tensor, reverse: bool, data_dtype: torch.dtype, ex) -> torch.Tensor:
    """scan_segments that also stores the chunk total into slot ex.rank of every
    rank's receive buffer and releases the flags (header: lasp2_scan_put). The
    epoch lives on the device (ex.ep): the put advances it, so this is safe to
    capture in a CUDA graph."""
    require_cuda(seg)
    b, h, nseg, d, _ = seg.shape
    total = torch.empty((b, h, d, d), dtype=seg.dtype, device=seg.device)
    if tuple(ex.recv.shape[2:]) != tuple(total.shape) or ex.recv.dtype != seg.dtype:
        raise ValueError(f"exchange buffer {tuple(ex.recv.shape)} {ex.recv.dtype} does not fit state "
                         f"{tuple(total.shape)} {seg.dtype}")
    ex.next_epoch()
    # back-pressure: every reader has acknowledged epoch e - 2 (= *ep - 1) before the put of e
    call("lasp2_exchange_wait", ptr(ex.acks), 0, ex.nranks, (1 << 64) - 1,
         ptr(ex.ep), stream_ptr())
    call("lasp2_scan_put", dtype_code(data_dtype), ptr(seg), ptr(total), b * h, nseg, d, int(reverse),
         ptr(ex.recv_table), ptr(ex.flag_table), ex.rank, ex.nranks, 0, ptr(ex.done), ptr(ex.ep), stream_ptr())
    return total


def exchange_fold(ex, mode: int, bound: int = 0) -> torch.Tensor:
    """Wait for the ranks a fold needs (header: lasp2_exchange_wait), fold this
    epoch's half of the rank-major receive buffer exactly like an all_gather
    result (lasp2_exchange_fold), then acknowledge the epoch to every writer
    (lasp2_exchange_ack). Every rank must call it once per exchange, also when it
    needs no state. All epoch values are read on the device."""
    lo, hi = {FOLD_PREFIX: (0, bound), FOLD_SUFFIX: (bound, ex.nranks), FOLD_FULL: (0, ex.nranks)}[mode]
    call("lasp2_exchange_wait", ptr(ex.flags), lo, hi, 0, ptr(ex.ep), stream_ptr())
    half = ex.recv[0]
    out = torch.empty(half.shape[1:], dtype=half.dtype, device=half.device)
    code = _lib.F64 if half.dtype == torch.float64 else _lib.F32
    call("lasp2_exchange_fold", code, ptr(ex.recv), half.numel(), ptr(ex.ep), ptr(out), ex.nranks, out.numel(), mode,
         bound, stream_ptr())
    exchange_ack(ex)
    return out


def exchange_ack(ex) -> None:
    """This rank is done with the current epoch's half (header: lasp2_exchange_ack)."""
    call("lasp2_exchange_ack", ptr(ex.ack_table), ex.rank, ex.nranks, 0, ptr(ex.ep), stream_ptr())


def causal_chunk_x(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, seg_states: torch.Tensor, ex, upto: int,
                   nseg: int, base_out: torch.Tensor | None = None) -> torch.Tensor:
    """causal_chunk whose base M_{1:upto} is folded in-kernel from the peer exchange
    (header: lasp2_causal_chunk_x, device epoch); acknowledges the epoch. bf16 only."""
    require_cuda(q, k, v, seg_states, base_out)
    slots, n, d = _slots(q)
    out = torch.empty_like(q)
    call("lasp2_causal_chunk_x", ptr(q), ptr(k), ptr(v), ptr(seg_states), ptr(ex.recv), ptr(ex.flags),
         0, upto, 0, 0, ptr(ex.ep), ex.recv[0].numel(), ptr(base_out), ptr(out), slots, n, d, nseg, 0, 0,
         stream_ptr())
    exchange_ack(ex)
    return out


def causal_chunk_gathered(q, k, v, seg_states, gathered: torch.Tensor, upto: int, nseg: int,
                          base_out: torch.Tensor | None = None) -> torch.Tensor:
    """causal_chunk whose base M_{1:upto} (ascending, copy-first) is folded in-kernel from
    a complete rank-major all_gather result [T, ...] (lasp2_causal_chunk_x, xflags NULL)."""
    require_cuda(q, k, v, seg_states, gathered, base_out)
    slots, n, d = _slots(q)
    out = torch.empty_like(q)
    call("lasp2_causal_chunk_x", ptr(q), ptr(k), ptr(v), ptr(seg_states), ptr(gathered), None, 0, upto, 0, 0, None, 0,
         ptr(base_out), ptr(out), slots, n, d, nseg, 0, 0, stream_ptr())
    return out


def dkdv_chunk_gathered(q, k, v, d_out, seg_states, gathered: torch.Tensor, start: int,
                        nseg: int) -> tuple[torch.Tensor, torch.Tensor]:
    """dkdv_chunk whose base (suffix of ranks >= start, descending) is folded in-kernel from
    a complete rank-major all_gather result (lasp2_dkdv_chunk_x, xflags NULL)."""
    require_cuda(q, k, v, d_out, seg_states, gathered)
    slots, n, d = _slots(q)
    dk, dv = torch.empty_like(k), torch.empty_like(v)
    call("lasp2_dkdv_chunk_x", ptr(q), ptr(k), ptr(v), ptr(d_out), ptr(seg_states), ptr(gathered), None, start,
         gathered.shape[0], 0, None, 0, ptr(dk), ptr(dv), slots, n, d, nseg, stream_ptr())
    return dk, dv


def dkdv_chunk_x(q, k, v, d_out, seg_states, ex, start: int, nseg: int) -> tuple[torch.Tensor, torch.Tensor]:
    """dkdv_chunk whose base (suffix of ranks >= start, descending) is folded in-kernel
    from the peer exchange (header: lasp2_dkdv_chunk_x, device epoch); acknowledges the epoch."""
    require_cuda(q, k, v, d_out, seg_states)
    slots, n, d = _slots(q)
    dk, dv = torch.empty_like(k), torch.empty_like(v)
    call("lasp2_dkdv_chunk_x", ptr(q), ptr(k), ptr(v), ptr(d_out), ptr(seg_states), ptr(ex.recv), ptr(ex.flags),
         start, ex.nranks, 0, ptr(ex.ep), ex.recv[0].numel(), ptr(dk), ptr(dv), slots, n, d, nseg, stream_ptr())
    exchange_ack(ex)
    return dk, dv


def fold(gathered: torch.Tensor, mode: int, bound: int = 0) -> torch.Tensor:
    """Ordered fold of rank-major gathered states [T, ...] (numerics.py:71-121)."""
    require_cuda(gathered)
    nstates = gathered.shape[0]
    out = torch.empty(gathered.shape[1:], dtype=gathered.dtype, device=gathered.device)
    code = _lib.F64 if gathered.dtype == torch.float64 else _lib.F32
    call("lasp2_fold_states", code, ptr(gathered), ptr(out), nstates, out.numel(), mode, bound, stream_ptr())
    return out


def prefix_states(gathered: torch.Tensor, upto: int) -> torch.Tensor:
    return fold(gathered, FOLD_PREFIX, upto)


def suffix_states(gathered: torch.Tensor, start: int) -> torch.Tensor:
    return fold(gathered, FOLD_SUFFIX, start)


def sum_states(gathered: torch.Tensor) -> torch.Tensor:
    return fold(gathered, FOLD_FULL, 0)


def causal_chunk(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, seg_states: torch.Tensor | None,
                 base: torch.Tensor | None, nseg: int, reverse: bool = False,
                 transpose_state: bool = False, out: torch.Tensor | None = None) -> torch.Tensor:
    """out_s = q_s S_s + sum_{i<=s} (q_s.k_i) v_i with S from base + segment states (see header)."""
    require_cuda(q, k, v, seg_states, base)
    if not (q.shape == k.shape == v.shape):
        raise ValueError(f"q/k/v shapes differ: {tuple(q.shape)} {tuple(k.shape)} {tuple(v.shape)}")
    slots, n, d = _slots(q)
    if out is None:
        out = torch.empty_like(q)
    call("lasp2_causal_chunk", dtype_code(q.dtype), ptr(q), ptr(k), ptr(v), ptr(seg_states), ptr(base), ptr(out),
         slots, n, d, nseg, int(reverse), int(transpose_state), stream_ptr())
    return out


def dq_chunk(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, d_out: torch.Tensor, fwd_seg: torch.Tensor | None,
             fwd_base: torch.Tensor | None, nseg: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Masked backward dQ plus the unscanned dM segment states Q_g^T dO_g (header: lasp2_dq_chunk)."""
    require_cuda(q, k, v, d_out, fwd_seg, fwd_base)
    if not (q.shape == k.shape == v.shape == d_out.shape):
        raise ValueError("q/k/v/d_out shapes differ")
    slots, n, d = _slots(q)
    b, h = q.shape[:2]
    gseg = torch.empty((b, h, nseg, d, d), dtype=state_dtype(q.dtype), device=q.device)
    dq = torch.empty_like(q)
    call("lasp2_dq_chunk", dtype_code(q.dtype), ptr(q), ptr(k), ptr(v), ptr(d_out), ptr(fwd_seg), ptr(fwd_base),
         ptr(gseg), ptr(dq), slots, n, d, nseg, stream_ptr())
    return dq, gseg


def dkdv_chunk(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, d_out: torch.Tensor,
               seg_states: torch.Tensor | None, base: torch.Tensor | None, nseg: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Masked backward dK, dV in one pass (header: lasp2_dkdv_chunk)."""
    require_cuda(q, k, v, d_out, seg_states, base)
    if not (q.shape == k.shape == v.shape == d_out.shape):
        raise ValueError("q/k/v/d_out shapes differ")
    slots, n, d = _slots(q)
    dk, dv = torch.empty_like(k), torch.empty_like(v)
    call("lasp2_dkdv_chunk", dtype_code(q.dtype), ptr(q), ptr(k), ptr(v), ptr(d_out), ptr(seg_states), ptr(base),
         ptr(dk), ptr(dv), slots, n, d, nseg, stream_ptr())
    return dk, dv


def backward_chunk(q, k, v, d_out, fwd_seg, fwd_total, fwd_base, bwd_seg, bwd_base, nseg: int):
    """(dq, dk, dv) of the masked chunk in one launch (header: lasp2_backward_chunk)."""
    require_cuda(q, k, v, d_out, fwd_seg, fwd_total, fwd_base, bwd_seg, bwd_base)
    slots, n, d = _slots(q)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    call("lasp2_backward_chunk", dtype_code(q.dtype), ptr(q), ptr(k), ptr(v), ptr(d_out), ptr(fwd_seg),
         ptr(fwd_total), ptr(fwd_base), ptr(bwd_seg), ptr(bwd_base), ptr(dq), ptr(dk), ptr(dv), slots, n, d, nseg,
         stream_ptr())
    return dq, dk, dv


def backward_chunk_fwd(q, k, v, d_out, fwd_seg, fwd_base, bwd_seg, bwd_total, bwd_base, nseg: int):
    """(dq, dk, dv) of the masked chunk in one launch, every CTA walking forwards
    (header: lasp2_backward_chunk_fwd); bwd_seg / bwd_total as the reverse scan leaves them."""
    require_cuda(q, k, v, d_out, fwd_seg, fwd_base, bwd_seg, bwd_total, bwd_base)
    slots, n, d = _slots(q)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    call("lasp2_backward_chunk_fwd", dtype_code(q.dtype), ptr(q), ptr(k), ptr(v), ptr(d_out), ptr(fwd_seg),
         ptr(fwd_base), ptr(bwd_seg), ptr(bwd_total), ptr(bwd_base), ptr(dq), ptr(dk), ptr(dv), slots, n, d, nseg,
         stream_ptr())
    return dq, dk, dv


def apply_state(x: torch.Tensor, m: torch.Tensor, transpose: bool = False,
                out: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
    """out (+)= x M or x M^T per slot (lasp2.py:150-165)."""
    require_cuda(x, m)
    slots, n, d = _slots(x)
    if m.shape != (*x.shape[:2], d, d):
        raise ValueError(f"state shape {tuple(m.shape)} does not match data {tuple(x.shape)}")
    if out is None:
        if accumulate:
            raise ValueError("accumulate needs an output tensor")
        out = torch.empty_like(x)
    call("lasp2_apply_state", dtype_code(x.dtype), ptr(x), ptr(m), ptr(out), slots, n, d, int(transpose),
         int(accumulate), stream_ptr())
    return out


def project(xs: list[torch.Tensor], ws: list[torch.Tensor], transpose: bool = False,
            out: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
    """out (+)= sum_i xs[i] op(ws[i]) per slot, op(W) = W or W^T, every W one [d, d] weight
    shared by all slots (header: lasp2_project; hybrid.py:136-151). len(xs) is 1 or 3."""
    import ctypes

    require_cuda(*xs, *ws)
    x0 = xs[0]
    slots, n, d = _slots(x0)
    if len(xs) != len(ws) or len(xs) not in (1, 3):
        raise ValueError("project takes one or three (input, weight) pairs")
    sd = state_dtype(x0.dtype)
    for x, w in zip(xs, ws):
        if x.shape != x0.shape or x.dtype != x0.dtype or not x.is_contiguous():
            raise ValueError(f"projection inputs differ: {tuple(x.shape)} {x.dtype}")
        if tuple(w.shape) != (d, d) or w.dtype != sd or not w.is_contiguous():
            raise ValueError(f"weight {tuple(w.shape)} {w.dtype} is not a contiguous ({d}, {d}) {sd} matrix")
    if out is None:
        if accumulate:
            raise ValueError("accumulate needs an output tensor")
        out = torch.empty_like(x0)
    xp = (ctypes.c_void_p * 3)(*[x.data_ptr() for x in xs])
    wp = (ctypes.c_void_p * 3)(*[w.data_ptr() for w in ws])
    call("lasp2_project", dtype_code(x0.dtype), ctypes.addressof(xp), ctypes.addressof(wp), len(xs), ptr(out), slots,
         n, d, int(transpose), int(accumulate), stream_ptr())
    return out


def state_apply(q: torch.Tensor, d_out: torch.Tensor, m: torch.Tensor, nseg: int) -> tuple[torch.Tensor, torch.Tensor]:
    """(dM segment states Q^T dO, dq = dO M^T) in one pass (header: lasp2_state_apply)."""
    require_cuda(q, d_out, m)
    slots, n, d = _slots(q)
    b, h = q.shape[:2]
    seg = torch.empty((b, h, nseg, d, d), dtype=state_dtype(q.dtype), device=q.device)
    dq = torch.empty_like(d_out)
    call("lasp2_state_apply", dtype_code(q.dtype), ptr(q), ptr(d_out), ptr(m), ptr(seg), ptr(dq), slots, n, d, nseg,
         stream_ptr())
    return seg, dq


def apply_state2(v: torch.Tensor, k: torch.Tensor, dm: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """(dk = v dM^T, dv = k dM) in one pass (header: lasp2_apply_state2)."""
    require_cuda(v, k, dm)
    slots, n, d = _slots(v)
    dk, dv = torch.empty_like(v), torch.empty_like(k)
    call("lasp2_apply_state2", dtype_code(v.dtype), ptr(v), ptr(k), ptr(dm), ptr(dk), ptr(dv), slots, n, d,
         stream_ptr())
    return dk, dv


_LOCAL_WS: OrderedDict[tuple[int, int], torch.Tensor] = OrderedDict()
_LOCAL_WS_MAX = 8  # streams with a cached workspace (least recently used dropped first)


def local_workspace(x: torch.Tensor) -> torch.Tensor:
    """Zero-initialised workspace of the world-of-one kernels, one per (device, stream).

    The kernels leave their grid-barrier words at zero, so the buffer is reused
    across calls on the same stream (the header's contract). At most
    _LOCAL_WS_MAX streams keep one: a dropped workspace was allocated on, and
    last used by, its own stream, so the caching allocator recycles it only
    behind that stream's queued kernels."""
    slots, n, d = _slots(x)
    need = int(_lib.load().lasp2_local_workspace_bytes(dtype_code(x.dtype), slots, n, d, sm_count(x.device)))
    if need < 0:
        raise ValueError(f"no world-of-one workspace for shape {tuple(x.shape)}")
    key = (x.device.index, torch.cuda.current_stream(x.device).cuda_stream)
    ws = _LOCAL_WS.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.zeros(max(need, 256), dtype=torch.uint8, device=x.device)
        _LOCAL_WS[key] = ws
    _LOCAL_WS.move_to_end(key)
    while len(_LOCAL_WS) > _LOCAL_WS_MAX:
        _LOCAL_WS.popitem(last=False)
    return ws


def nomask_forward_local(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """(out = q M, M = k^T v) of a world of one rank (header: lasp2_nomask_forward_local)."""
    require_cuda(q, k, v)
    if not (q.shape == k.shape == v.shape):
        raise ValueError(f"q/k/v shapes differ: {tuple(q.shape)} {tuple(k.shape)} {tuple(v.shape)}")
    slots, n, d = _slots(q)
    out = torch.empty_like(q)
    m_full = torch.empty((*q.shape[:2], d, d), dtype=state_dtype(q.dtype), device=q.device)
    ws = local_workspace(q)
    call("lasp2_nomask_forward_local", dtype_code(q.dtype), ptr(q), ptr(k), ptr(v), ptr(out), ptr(m_full), ptr(ws),
         ws.numel(), slots, n, d, stream_ptr())
    return out, m_full


def nomask_backward_local(q, k, v, d_out, m_full) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """(dq, dk, dv) of a world of one rank (header: lasp2_nomask_backward_local)."""
    require_cuda(q, k, v, d_out, m_full)
    if not (q.shape == k.shape == v.shape == d_out.shape):
        raise ValueError("q/k/v/d_out shapes differ")
    slots, n, d = _slots(q)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = local_workspace(q)
    call("lasp2_nomask_backward_local", dtype_code(q.dtype), ptr(q), ptr(k), ptr(v), ptr(d_out), ptr(m_full),
         ptr(dq), ptr(dk), ptr(dv), ptr(ws), ws.numel(), slots, n, d, stream_ptr())
    return dq, dk, dv


def nomask_forward_phase(q, k, v, m: torch.Tensor, phase: int, out: torch.Tensor | None = None):
    """Phase 1: m <- k^T v (this rank's chunk state); phase 2: out = q m with m the folded
    state (header: lasp2_nomask_forward_phase). Returns out (phase 2) or m (phase 1)."""
    require_cuda(k if phase == 1 else q, m)
    x = k if phase == 1 else q
    slots, n, d = _slots(x)
    if m.shape != (*x.shape[:2], d, d) or m.dtype != state_dtype(x.dtype) or not m.is_contiguous():
        raise ValueError(f"state {tuple(m.shape)} {m.dtype} does not match data {tuple(x.shape)}")
    if phase == 2 and out is None:
        out = torch.empty_like(q)
    ws = local_workspace(x)
    call("lasp2_nomask_forward_phase", dtype_code(x.dtype), ptr(q) if phase == 2 else 0, ptr(k) if phase == 1 else 0,
         ptr(v) if phase == 1 else 0, ptr(out) if phase == 2 else 0, ptr(m), ptr(ws), ws.numel(), slots, n, d, phase,
         stream_ptr(), label=f"lasp2_nomask_forward_phase{phase}")
    return out if phase == 2 else m


def nomask_forward_x(q, k, v, ex) -> tuple[torch.Tensor, torch.Tensor]:
    """(out, M_{1:T}) of one rank's unmasked forward in ONE launch with the state exchange
    fused in (header: lasp2_nomask_forward_x): the phase-1 reduction stores M_t into every
    rank's receive half, the kernel waits for every rank's flag, folds, acknowledges, and
    applies. The epoch lives on the device (ex.ep), so the call is graph-capturable."""
    require_cuda(q, k, v)
    slots, n, d = _slots(q)
    out = torch.empty_like(q)
    m = torch.empty((*q.shape[:2], d, d), dtype=state_dtype(q.dtype), device=q.device)
    _check_exchange(ex, m)
    ex.next_epoch()
    ws = local_workspace(q)
    call("lasp2_nomask_forward_x", ptr(q), ptr(k), ptr(v), ptr(out), ptr(m), ptr(ws), ws.numel(), slots, n, d,
         ptr(ex.recv), ptr(ex.recv_table), ptr(ex.flags), ptr(ex.flag_table), ptr(ex.acks), ptr(ex.ack_table),
         ex.rank, ex.nranks, ptr(ex.ep), stream_ptr(), label="lasp2_nomask_forward_x")
    return out, m


def nomask_backward_x(q, k, v, d_out, m_full, ex) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """(dq, dk, dv) of one rank's unmasked backward in ONE launch with the dM exchange fused
    in (header: lasp2_nomask_backward_x)."""
    require_cuda(q, k, v, d_out, m_full)
    slots, n, d = _slots(q)
    dq, dk, dv = torch.empty_like(d_out), torch.empty_like(v), torch.empty_like(k)
    dm = torch.empty_like(m_full)
    _check_exchange(ex, dm)
    ex.next_epoch()
    ws = local_workspace(q)
    call("lasp2_nomask_backward_x", ptr(q), ptr(k), ptr(v), ptr(d_out), ptr(m_full), ptr(dm), ptr(dq), ptr(dk),
         ptr(dv), ptr(ws), ws.numel(), slots, n, d, ptr(ex.recv), ptr(ex.recv_table), ptr(ex.flags),
         ptr(ex.flag_table), ptr(ex.acks), ptr(ex.ack_table), ex.rank, ex.nranks, ptr(ex.ep), stream_ptr(),
         label="lasp2_nomask_backward_x")
    return dq, dk, dv


def _check_exchange(ex, state: torch.Tensor) -> None:
    if tuple(ex.recv.shape[2:]) != tuple(state.shape) or ex.recv.dtype != state.dtype:
        raise ValueError(f"exchange buffer {tuple(ex.recv.shape)} {ex.recv.dtype} does not fit state "
                         f"{tuple(state.shape)} {state.dtype}")


def nomask_backward_phase1(q, d_out, m_full) -> tuple[torch.Tensor, torch.Tensor]:
    """(dq = d_out m_full^T, dm_t = q^T d_out) in one launch (header: lasp2_nomask_backward_phase)."""
    require_cuda(q, d_out, m_full)
    slots, n, d = _slots(q)
    dq = torch.empty_like(d_out)
    dm = torch.empty_like(m_full)
    ws = local_workspace(q)
    call("lasp2_nomask_backward_phase", dtype_code(q.dtype), ptr(q), 0, 0, ptr(d_out), ptr(m_full), ptr(dm), ptr(dq),
         0, 0, ptr(ws), ws.numel(), slots, n, d, 1, stream_ptr(), label="lasp2_nomask_backward_phase1")
    return dq, dm


def nomask_backward_phase2(v, k, dm) -> tuple[torch.Tensor, torch.Tensor]:
    """(dk = v dm^T, dv = k dm) with dm the folded dM (header: lasp2_nomask_backward_phase)."""
    require_cuda(v, k, dm)
    slots, n, d = _slots(v)
    if not dm.is_contiguous():
        dm = dm.contiguous()
    dk, dv = torch.empty_like(v), torch.empty_like(k)
    ws = local_workspace(v)
    call("lasp2_nomask_backward_phase", dtype_code(v.dtype), 0, ptr(k), ptr(v), 0, 0, ptr(dm), 0, ptr(dk), ptr(dv),
         ptr(ws), ws.numel(), slots, n, d, 2, stream_ptr(), label="lasp2_nomask_backward_phase2")
    return dk, dv


def softmax_forward(q: torch.Tensor, k_full: torch.Tensor, v_full: torch.Tensor, causal: bool, row_offset: int,
                    kv_tokens: int, kv_chunk: int, kv_rank_stride: int,
                    kv_start: int = 0) -> tuple[torch.Tensor, torch.Tensor]:
    """Softmax attention of a query chunk against (possibly rank-major) full K/V (oracle.py:136-139).
    kv_start > 0: the keys are [kv_start, kv_start + kv_tokens) of that layout (row_offset relative
    to kv_start; lasp2h_softmax_forward_range)."""
    require_cuda(q, k_full, v_full)
    slots, qn, d = _slots(q)
    out = torch.empty_like(q)
    lse = torch.empty(q.shape[:3], dtype=state_dtype(q.dtype), device=q.device)  # f64 data: f64 lse
    if kv_start or kv_tokens % kv_chunk:
        call("lasp2h_softmax_forward_range", dtype_code(q.dtype), ptr(q), ptr(k_full), ptr(v_full), ptr(out),
             ptr(lse), slots, qn, kv_tokens, d, int(causal), row_offset, kv_chunk, kv_rank_stride, kv_start,
             stream_ptr())
    else:
        call("lasp2h_softmax_forward", dtype_code(q.dtype), ptr(q), ptr(k_full), ptr(v_full), ptr(out), ptr(lse),
             slots, qn, kv_tokens, d, int(causal), row_offset, kv_chunk, kv_rank_stride, stream_ptr())
    return out, lse


def softmax_backward(q, k_full, v_full, out, lse, d_out, causal: bool, row_offset: int, kv_tokens: int,
                     kv_chunk: int, kv_rank_stride: int, grads: torch.Tensor, grad_rank_stride: int,
                     dv_offset: int) -> torch.Tensor:
    """dq plus full-length dk/dv contributions written into `grads` (oracle.py:142-158).

    dk contribution of key j lands at grads.view(-1)[(j//chunk)*grad_rank_stride + (slot*chunk + j%chunk)*d],
    dv at the same index + dv_offset.
    """
    return softmax_backward_acc(q, k_full, v_full, out, lse, d_out, causal, row_offset, kv_tokens, kv_chunk,
                                kv_rank_stride, grads, grad_rank_stride, dv_offset)[0]


def softmax_backward_acc(q, k_full, v_full, out, lse, d_out, causal: bool, row_offset: int, kv_tokens: int,
                         kv_chunk: int, kv_rank_stride: int, grads: torch.Tensor, grad_rank_stride: int,
                         dv_offset: int, key_range: bool = False,
                         kv_start: int = 0) -> tuple[torch.Tensor, torch.Tensor | None]:
    """softmax_backward that also returns the fp32 dQ accumulator the bf16 tensor-core
    path reduces into (None on the other paths, whose dq is already exact): partial
    dQs of one query chunk from several key ranges then add with one rounding.
    key_range: the keys are a sub-range of the softmax (lasp2h_softmax_backward_range)."""
    require_cuda(q, k_full, v_full, out, d_out, grads)
    slots, qn, d = _slots(q)
    dq = torch.empty_like(q)
    code = dtype_code(q.dtype)
    nbytes = int(_lib.load().lasp2h_softmax_scratch_bytes(code, slots, qn, kv_tokens, d))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=q.device)
    flat = grads.view(-1)
    args = (code, ptr(q), ptr(k_full), ptr(v_full), ptr(out), ptr(lse), ptr(d_out), ptr(dq), flat.data_ptr(),
            flat.data_ptr() + dv_offset * flat.element_size(), ptr(scratch), slots, qn, kv_tokens, d, int(causal),
            row_offset, kv_chunk, kv_rank_stride, grad_rank_stride)
    if key_range or kv_start:
        call("lasp2h_softmax_backward_range", *args, kv_start, stream_ptr())
    else:
        call("lasp2h_softmax_backward", *args, stream_ptr())
    acc = None
    if q.dtype == torch.bfloat16 and 8 <= d <= 128 and d % 8 == 0 and kv_chunk % 128 == 0:
        # tc_softmax_backward's scratch: delta [slots*qtok] (padded to 64) then dq_acc [slots][qtok][d] fp32
        off = ((slots * qn + 63) // 64) * 64
        acc = scratch.view(torch.float32)[off:off + slots * qn * d].view(q.shape)
    return dq, acc


def probe_gemm(a: torch.Tensor, b: torch.Tensor, a_mn: int, b_mn: bool) -> torch.Tensor:
    """D = op(A) op(B)^T for one 128^3 tile; a_mn 0/1 = K/MN-major smem A, 2 = A from TMEM."""
    require_cuda(a, b)
    d = torch.empty((128, 128), dtype=torch.float32, device=a.device)
    call("lasp2_debug_probe_gemm", ptr(a), ptr(b), ptr(d), int(a_mn), int(b_mn), stream_ptr())
    return d
