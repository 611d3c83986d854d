"""LASP-2 sequence-parallel linear attention on B200 (drop-in for laspsim.lasp2).

Same entry points, argument order and BHND layouts as the reference
(pkg/src/laspsim/lasp2.py), over torch CUDA tensors. Each rank owns one chunk
of C tokens; the only exchange per pass is one all_gather of the rank's d x d
memory states (lasp2.py:211/226/232/260/276).

Inside a GPU the chunk is split again into segments (one CTA per segment of a
(batch, head) slot), so every rank program is:

  forward  (masked, lasp2.py:219-243)
    seg = X^T Y per segment (K,V)        -> lasp2_segment_states
    scan seg (exclusive prefix), M_t     -> lasp2_scan_segments
    gathered = all_gather(M_t)           -> NCCL / emulated world
    P = prefix fold(gathered, t)         -> lasp2_fold_states
    O = mask(QK^T)V + Q (P + seg + ...)  -> lasp2_causal_chunk (tcgen05)
  backward (masked, lasp2.py:270-285)
    dM segments (Q, dO), suffix scan, all_gather(dM_t)   [in flight ...]
    dQ = causal(dO, V, K; S^T)                            [... during dQ]
    R = suffix fold(gathered, t+1)
    dK = anti-causal(V, dO, Q; G^T), dV = anti-causal(K, Q, dO; G)  -> lasp2_dkdv_chunk
    (or all three in one launch: lasp2_backward_chunk_fwd, MASKED_BWD_FUSED)

Precision follows the data dtype: bfloat16 runs the tcgen05/TMEM/TMA kernels
with fp32 states; float32 / float64 run the exact validation kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import comm, ops
from .shards import pack_slots, split_chunks, unpack_slots


def _as_device_tensor(x) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor):
        raise ValueError(f"expected a torch tensor or numpy array, got {type(x)}")
    if not x.is_cuda:
        if not torch.cuda.is_available():
            raise RuntimeError("the LASP-2 B200 path needs a CUDA device (no CPU fallback)")
        x = x.cuda()
    return x


@dataclass(frozen=True)
class ChunkedSequence:
    """Full q/k/v of shape (B, H, N, d) plus the chunk count T (lasp2.py:30-80)."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    chunks: int

    def __post_init__(self) -> None:
        # validate on the raw arrays first (lasp2.py:43-52), then move to the GPU
        arrs = [getattr(self, n) for n in ("q", "k", "v")]
        for name, arr in zip(("q", "k", "v"), arrs):
            if not isinstance(arr, (np.ndarray, torch.Tensor)):
                raise ValueError(f"{name} must be a torch tensor or numpy array, got {type(arr)}")
            if arr.ndim != 4:
                raise ValueError(f"{name} must be (batch, heads, tokens, dim), got {tuple(arr.shape)}")
        if not (tuple(arrs[0].shape) == tuple(arrs[1].shape) == tuple(arrs[2].shape)):
            raise ValueError(f"q/k/v shapes differ: {tuple(arrs[0].shape)}, {tuple(arrs[1].shape)}, "
                             f"{tuple(arrs[2].shape)}")
        if not (arrs[0].dtype == arrs[1].dtype == arrs[2].dtype):
            raise ValueError("q/k/v dtypes differ")
        n = arrs[0].shape[2]
        if self.chunks < 1 or n % self.chunks != 0:
            raise ValueError(f"chunk count {self.chunks} must divide sequence length {n}")
        for name, arr in zip(("q", "k", "v"), arrs):
            object.__setattr__(self, name, _as_device_tensor(arr))

    @property
    def batch(self) -> int:
        return self.q.shape[0]

    @property
    def heads(self) -> int:
        return self.q.shape[1]

    @property
    def seq_len(self) -> int:
        return self.q.shape[2]

    @property
    def dim(self) -> int:
        return self.q.shape[3]

    @property
    def chunk_len(self) -> int:
        return self.seq_len // self.chunks

    def chunk(self, t: int) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
        if not 0 <= t < self.chunks:
            raise ValueError(f"chunk index {t} outside [0, {self.chunks})")
        return (split_chunks(self.q, self.chunks)[t], split_chunks(self.k, self.chunks)[t],
                split_chunks(self.v, self.chunks)[t])


@dataclass
class GradientBundle:
    """Gradients w.r.t. q, k, v (oracle.py:41-47)."""

    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor


@dataclass
class ActivationCache:
    """Forward leftovers the backward may not recompute (lasp2.py:83-97).

    m_prefix = M_{1:t-1} (masked) or m_full = M_{1:T} (unmasked), exactly as in
    the reference. seg_prefix holds the rank-local exclusive segment prefixes of
    K^T V (the in-GPU analogue of the per-token states) so the backward never
    re-gathers or re-folds forward states; state_folds counts folds of
    gathered forward states (forward: 1, backward: 0 more).
    """

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    masked: bool
    m_prefix: torch.Tensor | None = None
    m_full: torch.Tensor | None = None
    state_folds: int = 0
    seg_prefix: torch.Tensor | None = None
    seg_total: torch.Tensor | None = None
    nseg: int = 1


@dataclass
class ForwardOutcome:
    outputs: list[torch.Tensor]
    caches: list[ActivationCache]
    run: comm.WorldRun


@dataclass
class BackwardOutcome:
    grads: list[GradientBundle]
    run: comm.WorldRun


@dataclass
class IterationOutcome:
    outputs: list[torch.Tensor]
    grads: list[GradientBundle]
    caches: list[ActivationCache]
    run: comm.WorldRun


# ---- per-rank programs ------------------------------------------------------

def _contig(*xs: torch.Tensor) -> list[torch.Tensor]:
    return [x.contiguous() for x in xs]


def _gather_states(ctx, m_t: torch.Tensor, tag: str, async_op: bool = False):
    """All-gather one (B,H,d,d) state per rank as pack_slots payload (shards.py:24-29)."""
    payload = pack_slots(m_t)
    return ctx.all_gather_async(payload, tag=tag) if async_op else ctx.all_gather(payload, tag=tag)


def _unpack_gathered(gathered: torch.Tensor, like: torch.Tensor) -> torch.Tensor:
    t = gathered.shape[0]
    return gathered.view(t, *like.shape)


# How a rank's chunk total reaches the other ranks. "collective": ctx.all_gather
# (NCCL all_gather_into_tensor on a side stream under torchrun). "peer": the scan
# kernel that produces M_t stores it straight into every rank's receive buffer
# (symmetric-memory peer addresses over NVLink) and releases a flag per rank;
# the fold waits on the flags it needs (lasp2_scan_put / lasp2_exchange_wait,
# SURVEY §8f.2). Both count one all_gather launch per exchange, same bytes. The
# exchange epoch lives on the device, so both are CUDA-graph capturable.
STATE_EXCHANGE = "collective"


def _peer(ctx, tag: str, like: torch.Tensor):
    if STATE_EXCHANGE != "peer" or ctx.sp_size == 1:
        return None
    fn = getattr(ctx, "peer_exchange", None)
    if fn is None:
        raise RuntimeError(f"STATE_EXCHANGE='peer' but {type(ctx).__name__} has no peer exchange")
    return fn(tag, like)  # None: this context keeps the all_gather (reported by the context)


# with the peer exchange, the bf16 chunk / dK-dV kernels wait for the ranks they need and
# fold the base in their own prologue (lasp2_causal_chunk_x / lasp2_dkdv_chunk_x): no wait or
# fold launch between the collective and its consumer. False: wait + fold kernels first.
PEER_FUSED_CONSUMER = True


def _fused_consumer(ctx, x: torch.Tensor) -> bool:
    # Only with one GPU per rank: in the threads-as-ranks world several ranks' kernels share
    # one GPU, and consumers spinning in-kernel could occupy every SM a producer still needs.
    d = x.shape[-1]
    return (PEER_FUSED_CONSUMER and getattr(ctx, "one_gpu_per_rank", False) and x.dtype == torch.bfloat16
            and 8 <= d <= 128 and d % 8 == 0)


# True: with the all_gather (NCCL) path too, the bf16 chunk / dK-dV kernels fold the
# prefix / suffix of the gathered states in their prologue (lasp2_causal_chunk_x /
# lasp2_dkdv_chunk_x with no flags), so no fold launch sits between the collective and
# its consumer. Off by default: every CTA of a slot then re-reads all T states of that
# slot (9-18x the fold kernel's L2 traffic, a few serial L2 latencies per CTA), which
# cost more than the fold launch it saves (cfg5 C = 8K per-rank step 0.170 -> 0.202 ms).
# The peer exchange keeps its fused consumers: there the prologue wait hides the exchange.
GATHERED_FUSED_CONSUMER = False


def _gathered_consumer(x: torch.Tensor) -> bool:
    d = x.shape[-1]
    return GATHERED_FUSED_CONSUMER and x.dtype == torch.bfloat16 and 8 <= d <= 128 and d % 8 == 0


def _share_total(ctx, seg: torch.Tensor, reverse: bool, data_dtype: torch.dtype, tag: str):
    """Scan the segment states; returns (chunk total, exchange handle or None)."""
    ex = _peer(ctx, tag, seg[:, :, 0])
    if ex is None:
        return ops.scan_segments(seg, reverse=reverse, data_dtype=data_dtype), None
    total = ops.scan_put(seg, reverse, data_dtype, ex)
    ctx.account_exchange(ex, tag)
    return total, ex


def _forward_nomask_rank(ctx, qc: torch.Tensor, kc: torch.Tensor,
                         vc: torch.Tensor) -> tuple[torch.Tensor, ActivationCache]:
    """O_t = Q_t M_{1:T} after one state all_gather (lasp2.py:208-216)."""
    qc, kc, vc = _contig(qc, kc, vc)
    if ctx.sp_size == 1 and LOCAL_FUSED:
        # world of one: the gather is the identity and sum_states a copy, so both
        # passes run as one persistent launch; the gather is still issued (1 launch,
        # as the reference accounts it)
        out, m_full = ops.nomask_forward_local(qc, kc, vc)
        _gather_states(ctx, m_full, "state")
        return out, ActivationCache(q=qc, k=kc, v=vc, masked=False, m_full=m_full, state_folds=1)
    if FLAT_PHASES:
        ex = _peer(ctx, "state", _state_like(kc))
        if ex is not None and _fused_consumer(ctx, qc):
            # one launch: phase 1, M_t stored into every rank's receive half, flag waits, the
            # full-sum fold and O = Q M_{1:T} (lasp2_nomask_forward_x)
            out, m_full = ops.nomask_forward_x(qc, kc, vc, ex)
            ctx.account_exchange(ex, "state")
            return out, ActivationCache(q=qc, k=kc, v=vc, masked=False, m_full=m_full, state_folds=1)
        # M_t from the persistent phase-1 launch (in-kernel ordered reduction), then the
        # exchange, then O = Q M_{1:T} as the dynamically scheduled phase-2 launch
        m_t = ops.nomask_forward_phase(qc, kc, vc, _state_like(kc), 1)
        if ex is not None:  # one-segment scan_put: a copy of M_t into every peer's buffer
            ops.scan_put(m_t.unsqueeze(2), False, kc.dtype, ex)
            ctx.account_exchange(ex, "state")
            m_full = ops.exchange_fold(ex, ops.FOLD_FULL)
        else:
            m_full = ops.sum_states(_unpack_gathered(_gather_states(ctx, m_t, "state"), m_t))
        out = ops.nomask_forward_phase(qc, kc, vc, m_full, 2)
        return out, ActivationCache(q=qc, k=kc, v=vc, masked=False, m_full=m_full, state_folds=1)
    nseg = ops.num_segments(kc)
    m_t, ex = _share_total(ctx, ops.segment_states(kc, vc, nseg), False, kc.dtype, "state")
    if ex is not None:
        m_full = ops.exchange_fold(ex, ops.FOLD_FULL)
        out = ops.apply_state(qc, m_full)
        return out, ActivationCache(q=qc, k=kc, v=vc, masked=False, m_full=m_full, state_folds=1)
    gathered = _unpack_gathered(_gather_states(ctx, m_t, "state"), m_t)
    m_full = ops.sum_states(gathered)
    out = ops.apply_state(qc, m_full)
    return out, ActivationCache(q=qc, k=kc, v=vc, masked=False, m_full=m_full, state_folds=1)


def _state_like(x: torch.Tensor) -> torch.Tensor:
    d = x.shape[-1]
    return torch.empty((*x.shape[:2], d, d), dtype=ops.state_dtype(x.dtype), device=x.device)


def _separate_inter(x: torch.Tensor) -> bool:
    """Validation modes (float32 / float64) keep the reference's grouping on every schedule:
    the intra-chunk term from a zero rank-level state, then `+= Q M_{1:t-1}` (and in the
    backward `+= dO M^T`, `+= V dM^T`, `+= K dM`) as separate passes (lasp2.py:236-240,
    :277-283). The sequential, overlap, LASP-1 ring and peer schedules then compute the
    same expression in the same order and agree bitwise (reference acceptance criteria 3
    and 8). bfloat16 folds the rank-level state into the chunk kernel's seed instead
    (one pass over the chunk, one rounding)."""
    return x.dtype != torch.bfloat16


def _forward_masked_rank(ctx, qc: torch.Tensor, kc: torch.Tensor, vc: torch.Tensor,
                         overlap: bool = False) -> tuple[torch.Tensor, ActivationCache]:
    """O_t = intra(Q_t, K_t, V_t) + Q_t M_{1:t-1} (lasp2.py:219-243).

    Sequential schedule: the gathered prefix is folded into the chunk kernel's
    initial state (one pass, one rounding). Overlap schedule: the chunk kernel
    runs while the all_gather is in flight and the inter term is added after
    the wait, Q_t M_{1:t-1} as a separate tensor-core pass (lasp2.py:224-230).
    """
    qc, kc, vc = _contig(qc, kc, vc)
    t = ctx.sp_position
    nseg = ops.num_segments(kc)
    seg = ops.segment_states(kc, vc, nseg)
    m_t, ex = _share_total(ctx, seg, False, kc.dtype, "state")
    if ex is not None:  # fused peer exchange: M_t is already on its way to every rank
        if _fused_consumer(ctx, qc) and not overlap:  # the chunk kernel waits and folds M_{1:t-1} itself
            m_prefix = torch.empty_like(m_t)
            ctx.mark("intra_start", f"chunk={t}")
            out = ops.causal_chunk_x(qc, kc, vc, seg, ex, t, nseg, base_out=m_prefix)
            ctx.mark("intra_end", f"chunk={t}")
        elif overlap:
            ctx.mark("intra_start", f"chunk={t}")
            out = ops.causal_chunk(qc, kc, vc, seg, None, nseg)
            ctx.mark("intra_end", f"chunk={t}")
            m_prefix = ops.exchange_fold(ex, ops.FOLD_PREFIX, t)
            if t > 0:
                ops.apply_state(qc, m_prefix, out=out, accumulate=True)
        else:
            m_prefix = ops.exchange_fold(ex, ops.FOLD_PREFIX, t)
            ctx.mark("intra_start", f"chunk={t}")
            out = ops.causal_chunk(qc, kc, vc, seg, m_prefix if t > 0 and not _separate_inter(qc) else None, nseg)
            ctx.mark("intra_end", f"chunk={t}")
            if t > 0 and _separate_inter(qc):
                ops.apply_state(qc, m_prefix, out=out, accumulate=True)
        return out, ActivationCache(q=qc, k=kc, v=vc, masked=True, m_prefix=m_prefix, state_folds=1,
                                    seg_prefix=seg, seg_total=m_t, nseg=nseg)
    if overlap:
        pending = _gather_states(ctx, m_t, "state", async_op=True)
        ctx.mark("intra_start", f"chunk={t}")
        out = ops.causal_chunk(qc, kc, vc, seg, None, nseg)
        ctx.mark("intra_end", f"chunk={t}")
        gathered = _unpack_gathered(pending.wait(), m_t)
        m_prefix = ops.prefix_states(gathered, t)
        if t > 0:
            ops.apply_state(qc, m_prefix, out=out, accumulate=True)
    else:
        gathered = _unpack_gathered(_gather_states(ctx, m_t, "state"), m_t)
        if _gathered_consumer(qc):  # the chunk kernel folds M_{1:t-1} from the gathered states itself
            m_prefix = torch.empty_like(m_t)
            ctx.mark("intra_start", f"chunk={t}")
            out = ops.causal_chunk_gathered(qc, kc, vc, seg, gathered, t, nseg, base_out=m_prefix)
        else:
            m_prefix = ops.prefix_states(gathered, t)
            ctx.mark("intra_start", f"chunk={t}")
            out = ops.causal_chunk(qc, kc, vc, seg, m_prefix if t > 0 and not _separate_inter(qc) else None, nseg)
            if t > 0 and _separate_inter(qc):
                ops.apply_state(qc, m_prefix, out=out, accumulate=True)
        ctx.mark("intra_end", f"chunk={t}")
    cache = ActivationCache(q=qc, k=kc, v=vc, masked=True, m_prefix=m_prefix, state_folds=1, seg_prefix=seg,
                            seg_total=m_t, nseg=nseg)
    return out, cache


def _require_cache(cache: ActivationCache, masked: bool) -> None:
    """lasp2.py:246-253."""
    if not isinstance(cache, ActivationCache):
        raise ValueError("backward needs the forward's ActivationCache")
    if cache.masked != masked:
        raise ValueError(f"cache was built masked={cache.masked}, backward wants {masked}")
    needed = cache.m_prefix if masked else cache.m_full
    if needed is None:
        raise ValueError("cache is missing its reduced state")
    if masked and cache.seg_prefix is None:
        raise ValueError("cache is missing its segment states")


def _backward_nomask_rank(ctx, cache: ActivationCache, d_out: torch.Tensor) -> GradientBundle:
    """One all_gather of Q^T dO; full-sum reduction (lasp2.py:256-267).

    When the all_gather is free (one rank) or cheap next to a pass over the
    chunk, dQ = dO M^T is fused into the dM segment pass (Q and dO read once);
    otherwise dQ runs while the collective is in flight. dK and dV share one pass.
    With FLAT_PHASES (default) both passes are the persistent flat kernels split
    around the exchange (lasp2_nomask_backward_phase).
    """
    _require_cache(cache, masked=False)
    (do,) = _contig(d_out)
    q = cache.q
    if ctx.sp_size == 1 and LOCAL_FUSED:
        dq, dk, dv = ops.nomask_backward_local(q, cache.k, cache.v, do, cache.m_full)
        _gather_states(ctx, cache.m_full, "state_grad")  # accounting only: identity at T = 1
        return GradientBundle(dq=dq, dk=dk, dv=dv)
    if FLAT_PHASES:
        ex = _peer(ctx, "state_grad", cache.m_full)
        if ex is not None and _fused_consumer(ctx, q):  # one launch, the dM exchange fused in
            dq, dk, dv = ops.nomask_backward_x(q, cache.k, cache.v, do, cache.m_full, ex)
            ctx.account_exchange(ex, "state_grad")
            return GradientBundle(dq=dq, dk=dk, dv=dv)
        # dQ and dM_t from the persistent phase-1 launch, the exchange, then dK, dV as phase 2
        dq, g_t = ops.nomask_backward_phase1(q, do, cache.m_full)
        if ex is not None:
            ops.scan_put(g_t.unsqueeze(2), False, q.dtype, ex)
            ctx.account_exchange(ex, "state_grad")
            dm_full = ops.exchange_fold(ex, ops.FOLD_FULL)
        else:
            dm_full = ops.sum_states(_unpack_gathered(_gather_states(ctx, g_t, "state_grad"), g_t))
        dk, dv = ops.nomask_backward_phase2(cache.v, cache.k, dm_full)
        return GradientBundle(dq=dq, dk=dk, dv=dv)
    unit_bytes = q.numel() * q.element_size()
    if ctx.sp_size == 1 or unit_bytes >= _FUSE_DQ_MIN_BYTES or STATE_EXCHANGE == "peer":
        nseg = ops.num_segments(q)
        gseg, dq = ops.state_apply(q, do, cache.m_full, nseg)
        g_t, ex = _share_total(ctx, gseg, False, q.dtype, "state_grad")
        if ex is not None:
            dm_full = ops.exchange_fold(ex, ops.FOLD_FULL)
            dk, dv = ops.apply_state2(cache.v, cache.k, dm_full)
            return GradientBundle(dq=dq, dk=dk, dv=dv)
        gathered = _unpack_gathered(_gather_states(ctx, g_t, "state_grad"), g_t)
    else:
        _, g_t, _ = ops.chunk_states(q, do)
        pending = _gather_states(ctx, g_t, "state_grad", async_op=True)
        dq = ops.apply_state(do, cache.m_full, transpose=True)  # independent of the collective
        gathered = _unpack_gathered(pending.wait(), g_t)
    dm_full = ops.sum_states(gathered)
    dk, dv = ops.apply_state2(cache.v, cache.k, dm_full)
    return GradientBundle(dq=dq, dk=dk, dv=dv)


# world of one rank: run the unmasked layer as one persistent launch per direction
# (lasp2_nomask_forward_local / _backward_local); False keeps the per-step kernels
LOCAL_FUSED = True

# T > 1 unmasked: the same persistent kernels split around the exchange (phase 1 ->
# M_t / dM_t, phase 2 after the fold; lasp2_nomask_*_phase); False keeps segment
# states + scan, apply_state / state_apply / apply_state2
FLAT_PHASES = True

# a bf16 chunk tensor of >= 256 MB takes >= ~40 us to stream, more than a
# state all_gather costs, so fusing dQ into the dM pass wins even with T > 1
_FUSE_DQ_MIN_BYTES = 256 << 20


def _backward_masked_rank(ctx, cache: ActivationCache, d_out: torch.Tensor) -> GradientBundle:
    """Masked backward (lasp2.py:270-285).

    One pass computes dQ (it needs only forward states) together with the dM
    segment states Q_g^T dO_g (lasp2_dq_chunk); their suffix scan gives M_t's
    gradient for the all_gather; after the descending suffix fold one pass
    computes dK and dV together (2-CTA clusters, Q/dO multicast).
    `MASKED_DQ_WITH_STATES = False` runs Q^T dO as its own pass with the gather
    in flight during dQ; `MASKED_BWD_FUSED = True` selects the single-launch
    dQ/dK/dV kernel (lasp2_backward_chunk_fwd).
    """
    _require_cache(cache, masked=True)
    t, world = ctx.sp_position, ctx.sp_size
    (do,) = _contig(d_out)
    q, k, v, nseg = cache.q, cache.k, cache.v, cache.nseg
    if MASKED_DQ_WITH_STATES and not MASKED_BWD_FUSED:
        # dq_s = sum_{i<=s}(do_s.v_i) k_i + do_s (M_{1:t-1} + local prefix)^T, and in the same
        # pass over (dO, V, K, Q) the dM segment states Q_g^T dO_g (lasp2.py:273-279)
        sep = _separate_inter(q)
        dq, gseg = ops.dq_chunk(q, k, v, do, cache.seg_prefix, cache.m_prefix if t > 0 and not sep else None, nseg)
        if t > 0 and sep:
            ops.apply_state(do, cache.m_prefix, transpose=True, out=dq, accumulate=True)
        g_t, ex = _share_total(ctx, gseg, True, q.dtype, "state_grad")
        if ex is not None and _fused_consumer(ctx, q):  # dK/dV kernel waits for ranks > t, folds their dM itself
            dk, dv = ops.dkdv_chunk_x(q, k, v, do, gseg, ex, t + 1, nseg)
            return GradientBundle(dq=dq, dk=dk, dv=dv)
        if ex is not None:  # every rank folds (and acknowledges) the exchange, the last one gets zeros
            r = ops.exchange_fold(ex, ops.FOLD_SUFFIX, t + 1)
            r = r if t < world - 1 else None
        else:
            gathered = _unpack_gathered(_gather_states(ctx, g_t, "state_grad"), g_t)
            if _gathered_consumer(q):  # the dK/dV kernel folds the suffix of ranks > t itself
                dk, dv = ops.dkdv_chunk_gathered(q, k, v, do, gseg, gathered, t + 1, nseg)
                return GradientBundle(dq=dq, dk=dk, dv=dv)
            r = ops.suffix_states(gathered, t + 1) if t < world - 1 else None
        dk, dv = ops.dkdv_chunk(q, k, v, do, gseg, None if sep else r, nseg)
        if sep and r is not None:
            ops.apply_state(v, r, transpose=True, out=dk, accumulate=True)
            ops.apply_state(k, r, out=dv, accumulate=True)
        return GradientBundle(dq=dq, dk=dk, dv=dv)
    gseg = ops.segment_states(q, do, nseg)
    g_t = ops.scan_segments(gseg, reverse=True, data_dtype=q.dtype)
    if MASKED_BWD_FUSED:
        gathered = _unpack_gathered(_gather_states(ctx, g_t, "state_grad"), g_t)
        r = ops.suffix_states(gathered, t + 1) if t < world - 1 else None
        dq, dk, dv = ops.backward_chunk_fwd(q, k, v, do, cache.seg_prefix, cache.m_prefix if t > 0 else None,
                                            gseg, g_t, r, nseg)
        return GradientBundle(dq=dq, dk=dk, dv=dv)
    pending = _gather_states(ctx, g_t, "state_grad", async_op=True)
    # dq_s = sum_{i<=s}(do_s.v_i) k_i + do_s (M_{1:t-1} + local prefix)^T   (overlaps the all_gather)
    dq = ops.causal_chunk(do, v, k, cache.seg_prefix, cache.m_prefix if t > 0 else None, nseg,
                          reverse=False, transpose_state=True)
    gathered = _unpack_gathered(pending.wait(), g_t)
    r = ops.suffix_states(gathered, t + 1) if t < world - 1 else None
    # dk_s = sum_{i>=s}(v_s.do_i) q_i + v_s G_s^T ; dv_s = sum_{i>=s}(k_s.q_i) do_i + k_s G_s  (one pass)
    dk, dv = ops.dkdv_chunk(q, k, v, do, gseg, r, nseg)
    return GradientBundle(dq=dq, dk=dk, dv=dv)


# single-launch dQ/dK/dV backward (lasp2_backward_chunk_fwd: three CTAs per segment
# walking forwards and sharing tiles through L2, 9 HBM units with the Q^T dO state
# pass instead of 11); off by default: its three 4-GEMM block chains per token block,
# not HBM, bound it, and it measures 2-3 % behind the dQ pass + dK/dV pair at cfg3
MASKED_BWD_FUSED = False

# masked backward default: the dQ pass also accumulates the dM segment states
# (lasp2_dq_chunk: Q, dO, V, K read once, 5 units instead of 2 + 4), so the dM
# all_gather follows the dQ pass; False restores the separate Q^T dO pass with
# the gather in flight during dQ
MASKED_DQ_WITH_STATES = True


# ---- world drivers ----------------------------------------------------------

def default_world(chunks: ChunkedSequence, **overrides) -> comm.WorldConfig:
    """One rank per chunk, element size from the data dtype (lasp2.py:290-293)."""
    overrides.setdefault("element_bytes", chunks.q.element_size())
    return comm.WorldConfig(world_size=chunks.chunks, sp_size=chunks.chunks, **overrides)


def _check_world(chunks: ChunkedSequence, cfg: comm.WorldConfig) -> None:
    if cfg.sp_size != chunks.chunks:
        raise ValueError(f"world sp_size {cfg.sp_size} != chunk count {chunks.chunks}")
    if cfg.element_bytes != chunks.q.element_size():
        raise ValueError(f"world element_bytes {cfg.element_bytes} does not match dtype {chunks.q.dtype}")


def _split_like(chunks: ChunkedSequence, full) -> list[torch.Tensor]:
    full = _as_device_tensor(full)
    if tuple(full.shape) != tuple(chunks.q.shape):
        raise ValueError(f"expected shape {tuple(chunks.q.shape)}, got {tuple(full.shape)}")
    return split_chunks(full.to(chunks.q.dtype), chunks.chunks)


def _spawn(chunks: ChunkedSequence, cfg: comm.WorldConfig | None, program,
           extra_args: list[tuple] | None = None) -> comm.WorldRun:
    cfg = cfg or default_world(chunks)
    _check_world(chunks, cfg)
    rank_args = []
    for rank in range(cfg.world_size):
        t = rank % cfg.sp_size  # DP replicas carry the same data (lasp2.py:316)
        qc, kc, vc = chunks.chunk(t)
        extra = extra_args[t] if extra_args is not None else ()
        rank_args.append((qc, kc, vc, *extra))
    return comm.world_spawn(cfg, program, rank_args, device=chunks.q.device)


def lasp2_forward_nomask(chunks: ChunkedSequence, cfg: comm.WorldConfig | None = None) -> ForwardOutcome:
    """lasp2.py:323-332."""
    run = _spawn(chunks, cfg, lambda ctx, qc, kc, vc: _forward_nomask_rank(ctx, qc, kc, vc))
    t = chunks.chunks
    return ForwardOutcome(outputs=[r[0] for r in run.results[:t]], caches=[r[1] for r in run.results[:t]], run=run)


def lasp2_forward_masked(chunks: ChunkedSequence, cfg: comm.WorldConfig | None = None,
                         overlap: bool = False) -> ForwardOutcome:
    """lasp2.py:335-344."""
    run = _spawn(chunks, cfg, lambda ctx, qc, kc, vc: _forward_masked_rank(ctx, qc, kc, vc, overlap=overlap))
    t = chunks.chunks
    return ForwardOutcome(outputs=[r[0] for r in run.results[:t]], caches=[r[1] for r in run.results[:t]], run=run)


def lasp2_overlap_schedule(chunks: ChunkedSequence, cfg: comm.WorldConfig | None = None) -> ForwardOutcome:
    """Masked forward with the collective in flight during intra compute (lasp2.py:347-355)."""
    return lasp2_forward_masked(chunks, cfg, overlap=True)


def _backward(chunks, d_out, caches, cfg, rank_fn) -> BackwardOutcome:
    if len(caches) != chunks.chunks:
        raise ValueError(f"expected {chunks.chunks} caches, got {len(caches)}")
    d_chunks = _split_like(chunks, d_out)
    run = _spawn(chunks, cfg, lambda ctx, qc, kc, vc, cache, dc: rank_fn(ctx, cache, dc),
                 extra_args=[(caches[t], d_chunks[t]) for t in range(chunks.chunks)])
    return BackwardOutcome(grads=run.results[:chunks.chunks], run=run)


def lasp2_backward_nomask(chunks: ChunkedSequence, d_out, caches: list[ActivationCache],
                          cfg: comm.WorldConfig | None = None) -> BackwardOutcome:
    """lasp2.py:358-371."""
    return _backward(chunks, d_out, caches, cfg, _backward_nomask_rank)


def lasp2_backward_masked(chunks: ChunkedSequence, d_out, caches: list[ActivationCache],
                          cfg: comm.WorldConfig | None = None) -> BackwardOutcome:
    """lasp2.py:374-387."""
    return _backward(chunks, d_out, caches, cfg, _backward_masked_rank)


def lasp2_iteration(chunks: ChunkedSequence, d_out, masked: bool, cfg: comm.WorldConfig | None = None,
                    overlap: bool = False) -> IterationOutcome:
    """Forward plus backward in one world: exactly 2 collective launches (lasp2.py:390-409)."""
    d_chunks = _split_like(chunks, d_out)

    def program(ctx, qc, kc, vc, dc):
        if masked:
            out, cache = _forward_masked_rank(ctx, qc, kc, vc, overlap=overlap)
            grad = _backward_masked_rank(ctx, cache, dc)
        else:
            out, cache = _forward_nomask_rank(ctx, qc, kc, vc)
            grad = _backward_nomask_rank(ctx, cache, dc)
        return out, grad, cache

    run = _spawn(chunks, cfg, program, extra_args=[(d_chunks[t],) for t in range(chunks.chunks)])
    t = chunks.chunks
    return IterationOutcome(outputs=[r[0] for r in run.results[:t]], grads=[r[1] for r in run.results[:t]],
                            caches=[r[2] for r in run.results[:t]], run=run)


# ---- per-rank entry points for torchrun (one process per GPU) ---------------

def rank_forward(ctx, qc: torch.Tensor, kc: torch.Tensor, vc: torch.Tensor, masked: bool = True,
                 overlap: bool = False) -> tuple[torch.Tensor, ActivationCache]:
    """The per-rank layer forward a model calls under torchrun (hybrid.py:171-175)."""
    if masked:
        return _forward_masked_rank(ctx, qc, kc, vc, overlap=overlap)
    return _forward_nomask_rank(ctx, qc, kc, vc)


def rank_backward(ctx, cache: ActivationCache, d_out: torch.Tensor) -> GradientBundle:
    """The per-rank layer backward (hybrid.py:193-197)."""
    if cache.masked:
        return _backward_masked_rank(ctx, cache, d_out)
    return _backward_nomask_rank(ctx, cache, d_out)


__all__ = [
    "ActivationCache", "BackwardOutcome", "ChunkedSequence", "ForwardOutcome", "GradientBundle", "IterationOutcome",
    "default_world", "lasp2_backward_masked", "lasp2_backward_nomask", "lasp2_forward_masked",
    "lasp2_forward_nomask", "lasp2_iteration", "lasp2_overlap_schedule", "rank_backward", "rank_forward",
    "pack_slots", "unpack_slots",
]


# ---- per-slot kernels under the reference names (lasp2.py:126-203) ----------

def chunk_state(kc: torch.Tensor, vc: torch.Tensor) -> torch.Tensor:
    """M = K^T V per slot, (B, H, d, d) (lasp2.py:130-137)."""
    kc, vc = _contig(_as_device_tensor(kc), _as_device_tensor(vc))
    return ops.chunk_states(kc, vc)[1]


def chunk_state_grad(qc: torch.Tensor, d_out: torch.Tensor) -> torch.Tensor:
    """G = Q^T dO per slot (lasp2.py:140-147)."""
    qc, do = _contig(_as_device_tensor(qc), _as_device_tensor(d_out))
    return ops.chunk_states(qc, do)[1]


def apply_state(xc: torch.Tensor, m: torch.Tensor) -> torch.Tensor:
    """X @ M per slot (lasp2.py:150-156)."""
    xc, m = _contig(_as_device_tensor(xc), _as_device_tensor(m))
    return ops.apply_state(xc, m)


def apply_state_t(xc: torch.Tensor, m: torch.Tensor) -> torch.Tensor:
    """X @ M^T per slot (lasp2.py:159-165)."""
    xc, m = _contig(_as_device_tensor(xc), _as_device_tensor(m))
    return ops.apply_state(xc, m, transpose=True)


def intra_forward(qc: torch.Tensor, kc: torch.Tensor, vc: torch.Tensor) -> torch.Tensor:
    """Causal attention within the chunk (lasp2.py:168-174 / oracle.py:50-62)."""
    qc, kc, vc = _contig(*map(_as_device_tensor, (qc, kc, vc)))
    seg, _, nseg = ops.chunk_states(kc, vc)
    return ops.causal_chunk(qc, kc, vc, seg, None, nseg)


def intra_forward_left_product(qc: torch.Tensor, kc: torch.Tensor, vc: torch.Tensor) -> torch.Tensor:
    """[(Q K^T) o Psi] V (lasp2.py:177-186): the blocked form the kernel evaluates."""
    return intra_forward(qc, kc, vc)


def intra_backward(qc: torch.Tensor, kc: torch.Tensor, vc: torch.Tensor, d_out: torch.Tensor) -> GradientBundle:
    """Gradients of the masked intra-chunk term (lasp2.py:189-203)."""
    q, k, v, do = _contig(*map(_as_device_tensor, (qc, kc, vc, d_out)))
    seg, _, nseg = ops.chunk_states(k, v)
    gseg = ops.segment_states(q, do, nseg)
    ops.scan_segments(gseg, reverse=True, data_dtype=q.dtype)
    dq = ops.causal_chunk(do, v, k, seg, None, nseg, reverse=False, transpose_state=True)
    dk, dv = ops.dkdv_chunk(q, k, v, do, gseg, None, nseg)
    return GradientBundle(dq=dq, dk=dk, dv=dv)
