"""Rank-ordered state folds with the reference's list interface (numerics.py:60-121).

Drop-in names for callers of ``laspsim.numerics`` (hybrid.py:23, cli.py): the
states are a rank-ordered sequence of same-shaped CUDA tensors (or one stacked
[T, ...] tensor, the all_gather layout) and every fold runs as one
``lasp2_fold_states`` launch with the reference's order and seeding:

* prefix: copy states[0], add states[1..upto-1] ascending; upto = 0 -> zeros;
* suffix: copy states[n-1], add states[n-2..start] descending; start = n -> zeros;
* full: the ascending prefix over all n.

Never starting from a zero accumulator keeps -0.0 entries (numerics.py:6-8),
so these agree bitwise with the reference's loops on the same f64 data.
"""
from __future__ import annotations

from collections.abc import Sequence

import torch

from . import ops


def _stacked(states: Sequence[torch.Tensor] | torch.Tensor) -> torch.Tensor:
    """Validate like numerics.py:60-66 and return the rank-major [n, ...] stack."""
    if isinstance(states, torch.Tensor):
        if states.ndim < 1 or states.shape[0] == 0:
            raise ValueError("state list must be non-empty")
        return states.contiguous()
    if len(states) == 0:
        raise ValueError("state list must be non-empty")
    shape = tuple(states[0].shape)
    for i, s in enumerate(states):
        if tuple(s.shape) != shape:
            raise ValueError(f"state {i} has shape {tuple(s.shape)}, expected {shape}")
        if s.dtype != states[0].dtype:
            raise ValueError(f"state {i} has dtype {s.dtype}, expected {states[0].dtype}")
    return torch.stack(list(states))


def _fold_dtype_ok(x: torch.Tensor) -> None:
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"states are float32 or float64 (the fold dtypes), got {x.dtype}")


def prefix_sum_states(states: Sequence[torch.Tensor] | torch.Tensor, upto: int) -> torch.Tensor:
    """Sum of states[0:upto] folded in ascending order (numerics.py:69-89)."""
    x = _stacked(states)
    n = x.shape[0]
    if not 0 <= upto <= n:
        raise ValueError(f"upto={upto} outside [0, {n}]")
    _fold_dtype_ok(x)
    return ops.prefix_states(x, upto)


def suffix_sum_states(states: Sequence[torch.Tensor] | torch.Tensor, start: int) -> torch.Tensor:
    """Sum of states[start:] folded in descending order (numerics.py:92-116)."""
    x = _stacked(states)
    n = x.shape[0]
    if not 0 <= start <= n:
        raise ValueError(f"start={start} outside [0, {n}]")
    _fold_dtype_ok(x)
    return ops.suffix_states(x, start)


def sum_states(states: Sequence[torch.Tensor] | torch.Tensor) -> torch.Tensor:
    """Full ascending-order fold over all states (numerics.py:119-121)."""
    x = _stacked(states)
    return prefix_sum_states(x, x.shape[0])
