"""ctypes binding of the C-ABI library (include/lasp2_b200.h).

The library is the product: there is no Python or CPU fallback. If the
shared object is missing or a CUDA device is absent, every compute call raises.
"""
from __future__ import annotations

import ctypes
import re
import threading
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "liblasp2_b200.so"
HEADER = Path(__file__).resolve().parent.parent / "include" / "lasp2_b200.h"

F32, F64, BF16 = 0, 1, 2
FOLD_PREFIX, FOLD_SUFFIX, FOLD_FULL = 0, 1, 2

_i64 = ctypes.c_int64
_int = ctypes.c_int
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64

# name -> (restype, argtypes); must match include/lasp2_b200.h
SIGNATURES = {
    "lasp2_version": (_int, []),
    "lasp2_last_error": (ctypes.c_char_p, []),
    "lasp2_num_segments": (_int, [_int, _i64, _i64, _int, _int]),
    "lasp2_segment_states": (_int, [_int, _vp, _vp, _vp, _i64, _i64, _int, _int, _vp]),
    "lasp2_scan_segments": (_int, [_int, _vp, _vp, _i64, _int, _int, _int, _vp]),
    "lasp2_fold_states": (_int, [_int, _vp, _vp, _int, _i64, _int, _int, _vp]),
    "lasp2_causal_chunk": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _int, _int, _int, _int, _vp]),
    "lasp2_scan_put": (_int, [_int, _vp, _vp, _i64, _int, _int, _int, _vp, _vp, _int, _int, _u64, _vp, _vp, _vp]),
    "lasp2_exchange_wait": (_int, [_vp, _int, _int, _u64, _vp, _vp]),
    "lasp2_exchange_ack": (_int, [_vp, _int, _int, _u64, _vp, _vp]),
    "lasp2_exchange_fold": (_int, [_int, _vp, _i64, _vp, _vp, _int, _i64, _int, _int, _vp]),
    "lasp2_causal_chunk_x": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _int, _int, _int, _u64, _vp, _i64, _vp, _vp, _i64,
                                    _i64, _int, _int, _int, _int, _vp]),
    "lasp2_dkdv_chunk_x": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _int, _int, _u64, _vp, _i64, _vp, _vp, _i64,
                                  _i64, _int, _int, _vp]),
    "lasp2_dq_chunk": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _int, _int, _vp]),
    "lasp2_dkdv_chunk": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _int, _int, _vp]),
    "lasp2_project": (_int, [_int, _vp, _vp, _int, _vp, _i64, _i64, _int, _int, _int, _vp]),
    "lasp2_state_apply": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _int, _int, _vp]),
    "lasp2_apply_state2": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _int, _vp]),
    "lasp2_backward_chunk": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64,
                                    _int, _int, _vp]),
    "lasp2_backward_chunk_fwd": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64,
                                        _i64, _int, _int, _vp]),
    "lasp2_nomask_forward_x": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp,
                                      _vp, _vp, _int, _int, _vp, _vp]),
    "lasp2_nomask_backward_x": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int,
                                       _vp, _vp, _vp, _vp, _vp, _vp, _int, _int, _vp, _vp]),
    "lasp2_apply_state": (_int, [_int, _vp, _vp, _vp, _i64, _i64, _int, _int, _int, _vp]),
    "lasp2_local_workspace_bytes": (_i64, [_int, _i64, _i64, _int, _int]),
    "lasp2_nomask_forward_local": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _vp]),
    "lasp2_nomask_backward_local": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64,
                                           _int, _vp]),
    "lasp2_nccl_unique_id": (_int, [_vp]),
    "lasp2_nccl_comm_init": (_int, [_vp, _int, _vp, _int]),
    "lasp2_nccl_comm_destroy": (_int, [_vp]),
    "lasp2_state_allgather": (_int, [_vp, _int, _vp, _vp, _i64, _vp]),
    "lasp2h_kv_allgather": (_int, [_vp, _int, _vp, _vp, _vp, _vp, _i64, _vp]),
    "lasp2h_grad_reduce_scatter": (_int, [_vp, _int, _vp, _vp, _i64, _vp]),
    "lasp2_nomask_forward_phase": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp]),
    "lasp2_nomask_backward_phase": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64,
                                           _i64, _int, _int, _vp]),
    "lasp2h_softmax_forward_range": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _i64,
                                            _i64, _i64, _i64, _vp]),
    "lasp2h_softmax_forward": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _i64, _i64, _i64,
                                      _vp]),
    "lasp2h_softmax_backward": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int,
                                       _int, _i64, _i64, _i64, _i64, _vp]),
    "lasp2h_softmax_backward_range": (_int, [_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64,
                                             _i64, _int, _int, _i64, _i64, _i64, _i64, _i64, _vp]),
    "lasp2h_softmax_scratch_bytes": (_i64, [_int, _i64, _i64, _i64, _int]),
    "lasp2_gen_slots": (_int, [_int, _u64, _vp, _vp, _i64, _i64, _i64, _i64, _vp]),
    "lasp2_debug_probe_gemm": (_int, [_vp, _vp, _vp, _int, _int, _vp]),
    "lasp2_debug_trace": (_int, [_vp]),
}

_lock = threading.Lock()
_lib = None


class LaspError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


def header_symbols() -> list[str]:
    """Function names declared in include/lasp2_b200.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(lasp2h?_\w+)\s*\(", text, re.M)))


def load() -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise FileNotFoundError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2502_07563_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class _Profiler:
    """Optional per-entry-point device timing and launch counting (bench.py).

    When enabled, every C-ABI compute call is bracketed by CUDA events on the
    stream it is enqueued on, so per-kernel durations are measured live inside
    a timed region without a profiler attached.
    """

    def __init__(self) -> None:
        self.enabled = False
        self.launches = 0
        self.events: dict[str, list] = {}

    def reset(self, enabled: bool) -> None:
        self.enabled = enabled
        self.launches = 0
        self.events = {}

    def durations_ms(self) -> dict[str, list[float]]:
        return {k: [a.elapsed_time(b) for a, b in v] for k, v in self.events.items()}


PROFILER = _Profiler()
# kernels launched per call of each entry point (for gpu_launches accounting)
KERNELS_PER_CALL = {"lasp2h_softmax_backward": 4,  # bf16 tc path: delta, memset, main, finalize
                    "lasp2h_softmax_backward_range": 4}
_NO_LAUNCH = {"lasp2_version", "lasp2_last_error", "lasp2_num_segments", "lasp2h_softmax_scratch_bytes",
              "lasp2_local_workspace_bytes",
              "lasp2_debug_trace",
              # NCCL's kernels, not this library's
              "lasp2_nccl_unique_id", "lasp2_nccl_comm_init", "lasp2_nccl_comm_destroy", "lasp2_state_allgather",
              "lasp2h_kv_allgather", "lasp2h_grad_reduce_scatter"}


def call(name: str, *args, label: str | None = None) -> int:
    """Call a C-ABI entry point; raise on a non-zero status. `label` names the call in
    the profiler when one entry point launches different kernels (e.g. the two phases
    of lasp2_nomask_*_phase)."""
    lib = load()
    prof = PROFILER
    if prof.enabled and name not in _NO_LAUNCH:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        status = getattr(lib, name)(*args)
        b.record()
        prof.events.setdefault(label or name, []).append((a, b))
        prof.launches += KERNELS_PER_CALL.get(name, 1)
    else:
        status = getattr(lib, name)(*args)
    if status != 0:
        msg = lib.lasp2_last_error().decode()
        if status == 1:
            raise ValueError(f"{name}: {msg}")
        raise LaspError(f"{name} failed (status {status}): {msg}")
    return status


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return F32
    if dt == torch.float64:
        return F64
    if dt == torch.bfloat16:
        return BF16
    raise ValueError(f"unsupported dtype {dt}; expected float64, float32 or bfloat16")


def state_dtype(dt: torch.dtype) -> torch.dtype:
    """Memory states / gathered payloads: f64 for f64 data, else f32."""
    return torch.float64 if dt == torch.float64 else torch.float32


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda(*tensors: torch.Tensor) -> None:
    for t in tensors:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("LASP-2 B200 kernels need CUDA tensors (no CPU fallback)")
        if not t.is_contiguous():
            raise ValueError("LASP-2 B200 kernels need contiguous BHND tensors")
