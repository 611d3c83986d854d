"""Verify / bench / cost-table harness over the B200 drivers, with the
reference CLI's run configuration, check records and CSV tables
(reference cli.py:46-50 columns, :120-196 RunConfig / Check, :339-498
per-method checks, :654-810 verify / bench / costmodel).

    python -m paper_2502_07563_b200.harness verify --method lasp2 --seq-len 64 --chunks 4
    python -m paper_2502_07563_b200.harness bench --method lasp2 --precision bf16 --seq-len 65536 --dim 128 --heads 16
    python -m paper_2502_07563_b200.harness costmodel --world 8

The checks compare the GPU drivers with float64 restatements evaluated here
with torch on the device: the left-product form [(QK^T) * Psi] V for linear
attention, masked softmax attention, the exclusive-prefix ring form
(cli.py:244-278), the L/N layer stack, and autograd for their gradients. They
are independent of the repo's test oracle (oracle/), which stays test-only.

Deviations from the reference harness, each because the arithmetic runs on a
GPU instead of through one numpy BLAS:
* checks the reference states as bitwise (tolerance 0: one-chunk runs vs the
  serial oracle, LASP-1 vs LASP-2, the ring's exclusive-prefix form) use the
  forward / gradient tolerance of the precision instead;
* precision "bf16" (the tensor-core path) is added; its errors are normalised,
  max|got - ref| / max|ref| per tensor, against 1e-2 (SURVEY §8a note P).
  A bf16 L/N stack is only checkable for well-conditioned patterns: an
  unnormalised L layer (no norm, as in the reference) gives the next softmax
  logits of size ~N, where bf16 rounding flips row maxima;
* method "oracle" (the reference checking its own serial oracles) is not a
  B200 path and is refused.
``simulated_time`` is the threads-as-ranks world's simulated clock
(comm.py); ``wall_time_ns`` includes input generation like the reference's.
"""
from __future__ import annotations

import argparse
import csv
import hashlib
import itertools
import json
import math
import sys
import time
from dataclasses import asdict, dataclass

import torch

from . import __version__, comm, costmodel
from .datagen import gen_slots_device
from .hybrid import ModelSpec, hybrid_iteration, layer_weights
from .lasp1 import lasp1_iteration
from .lasp2 import ChunkedSequence, lasp2_iteration
from .standard_sp import cp_iteration

METHODS = ("lasp1", "lasp2", "lasp2h", "cp")
PRECISIONS = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}

BENCH_COLUMNS = ["method", "N", "T", "W", "d", "H", "B", "masked",
                 "steps", "launches", "bytes", "simulated_time", "wall_time_ns"]
COST_COLUMNS = ["method", "W", "T", "B", "H", "d", "element_bytes", "iterations",
                "steps_per_iteration", "traffic_per_step_bytes",
                "state_param_count", "total_traffic_bytes"]

_FD_MAX_N = 16
_FD_MAX_D = 8

_TOLS = {  # cli.py:56-63, plus bf16 (normalised errors)
    "f64": {"forward": 1e-10, "forward_softmax": 1e-12, "grad_serial": 1e-12, "grad_softmax": 1e-10,
            "fd": 1e-6, "stack": 1e-9},
    "f32": {"forward": 1e-3, "forward_softmax": 1e-3, "grad_serial": 1e-3, "grad_softmax": 1e-3,
            "fd": None, "stack": 1e-2},
    "bf16": {"forward": 1e-2, "forward_softmax": 1e-2, "grad_serial": 1e-2, "grad_softmax": 1e-2,
             "fd": None, "stack": 1e-2},
}


class UsageError(Exception):
    """Bad flags, config keys or parameter combinations; exit code 2 (cli.py:66-67)."""


_TRUE, _FALSE = frozenset({"true", "1", "yes"}), frozenset({"false", "0", "no"})


def _parse_bool(text: str) -> bool:
    word = text.strip().lower()
    if word in _TRUE or word in _FALSE:
        return word in _TRUE
    raise ValueError(text)


# key -> (parser, what the value must look like); keys accept '-' or '_' and leading dashes
_KEY_TYPES = {
    **{k: (int, "an integer") for k in ("seq_len", "chunks", "world", "dim", "heads", "batch", "seed",
                                        "element_bytes", "iterations")},
    **{k: (float, "a number") for k in ("latency_per_launch", "latency_per_byte")},
    **{k: (str, "a string") for k in ("method", "pattern", "precision")},
    "masked": (_parse_bool, "true or false"),
}


def _coerce(key: str, value):
    """(normalised key, typed value) of one flag or config-file entry (cli.py:70-117)."""
    name = key.strip().lstrip("-").replace("-", "_")
    if name not in _KEY_TYPES:
        raise UsageError(f"unknown configuration key {key.strip()!r}")
    parse, expected = _KEY_TYPES[name]
    if not isinstance(value, str):
        return name, value
    try:
        return name, parse(value)
    except ValueError:
        raise UsageError(f"expected {expected}, got {value!r}") from None


@dataclass(frozen=True)
class RunConfig:
    """One fully resolved run (cli.py:120-180)."""

    method: str = "lasp2"
    seq_len: int = 64
    chunks: int = 4
    world: int | None = None
    dim: int = 8
    heads: int = 1
    batch: int = 1
    masked: bool = True
    pattern: str = ""
    precision: str = "f64"
    seed: int = 0
    latency_per_launch: float = 10.0
    latency_per_byte: float = 1.0 / 1024.0

    def __post_init__(self) -> None:
        if self.method == "oracle":
            raise UsageError("method 'oracle' checks the reference's own serial oracles; "
                             "the B200 build keeps its oracle in tests (oracle/)")
        if self.method not in METHODS:
            raise UsageError(f"unknown method {self.method!r}; choose from {METHODS}")
        if self.precision not in PRECISIONS:
            raise UsageError(f"unknown precision {self.precision!r}; choose from {tuple(PRECISIONS)}")
        for name in ("seq_len", "chunks", "dim", "heads", "batch"):
            if getattr(self, name) < 1:
                raise UsageError(f"{name} must be positive, got {getattr(self, name)}")
        if self.seq_len % self.chunks != 0:
            raise UsageError(f"chunks {self.chunks} must divide seq_len {self.seq_len}")
        if self.world is None:
            object.__setattr__(self, "world", self.chunks)
        if self.world % self.chunks != 0:
            raise UsageError(f"chunks {self.chunks} must divide world {self.world}")
        if self.method == "lasp2h":
            if not self.pattern.replace(" ", ""):
                raise UsageError("method lasp2h needs a nonempty --pattern")
        elif self.pattern:
            raise UsageError(f"--pattern applies only to lasp2h, not {self.method}")
        if self.latency_per_launch < 0 or self.latency_per_byte < 0:
            raise UsageError("latency parameters must be nonnegative")

    @property
    def dtype(self) -> torch.dtype:
        return PRECISIONS[self.precision]

    @property
    def element_bytes(self) -> int:
        return torch.empty(0, dtype=self.dtype).element_size()

    def world_config(self) -> comm.WorldConfig:
        return comm.WorldConfig(world_size=self.world, sp_size=self.chunks, element_bytes=self.element_bytes,
                                latency_per_launch=self.latency_per_launch,
                                latency_per_byte=self.latency_per_byte)

    def config_hash(self) -> str:
        return hashlib.sha256(json.dumps(asdict(self), sort_keys=True).encode("utf-8")).hexdigest()


@dataclass
class Check:
    """One named invariant: observed deviation against its tolerance (cli.py:183-196)."""

    name: str
    max_error: float
    tolerance: float

    @property
    def passed(self) -> bool:
        return self.max_error <= self.tolerance

    def as_dict(self) -> dict:
        return {"name": self.name, "max_error": self.max_error, "tolerance": self.tolerance,
                "passed": self.passed}


# ---- float64 restatements on the device -----------------------------------------

def _linear_full(q, k, v, causal):
    s = q @ k.transpose(-1, -2)
    if causal:
        s = torch.tril(s)
    return s @ v


def _softmax_full(q, k, v, causal):
    s = (q @ k.transpose(-1, -2)) / math.sqrt(q.shape[-1])
    if causal:
        n = q.shape[-2]
        s = s.masked_fill(torch.ones(n, n, dtype=torch.bool, device=q.device).triu(1), float("-inf"))
    return torch.softmax(s, dim=-1) @ v


def _exclusive_prefix_forward(q, k, v, chunks):
    """What the ring computes without a mask: O_t = Q_t (sum of earlier chunk states) (cli.py:244-255)."""
    qs, ks, vs = (x.chunk(chunks, dim=2) for x in (q, k, v))
    states = torch.stack([kc.transpose(-1, -2) @ vc for kc, vc in zip(ks, vs)])
    prefix = torch.cumsum(states, 0) - states
    return torch.cat([qc @ prefix[t] for t, qc in enumerate(qs)], dim=2)


def _grads(fn, arrays, d_out):
    xs = [a.detach().clone().requires_grad_(True) for a in arrays]
    return torch.autograd.grad(fn(*xs), xs, d_out)


def _fd_grads(fn, arrays, d_out, h=1e-6):
    """Central differences of sum(fn(...) * d_out) (oracle.py finite_diff_grad)."""
    out = []
    for i in range(len(arrays)):
        x = arrays[i].clone()
        g = torch.empty_like(x)
        flat, gf = x.view(-1), g.view(-1)
        for j in range(flat.numel()):
            old = flat[j].item()
            vals = []
            for delta in (h, -h):
                flat[j] = old + delta
                args = list(arrays)
                args[i] = x
                vals.append(float((fn(*args) * d_out).sum()))
            flat[j] = old
            gf[j] = (vals[0] - vals[1]) / (2 * h)
        out.append(g)
    return out


def _cat(xs) -> torch.Tensor:
    return torch.cat([x.double() for x in xs], dim=2)


def _error(got: torch.Tensor, ref: torch.Tensor, precision: str, kind: str) -> float:
    """kind 'abs': max |got - ref| (cli.py:294-295); 'rel': element-wise with a
    max(1, |ref|) floor (oracle.py relative_error). bf16: normalised error."""
    if got.numel() == 0:
        return 0.0
    diff = (got.double() - ref.double()).abs()
    if precision == "bf16":
        scale = ref.double().abs().max().item()
        return diff.max().item() / scale if scale > 0 else diff.max().item()
    if kind == "abs":
        return diff.max().item()
    return (diff / ref.double().abs().clamp_min(1.0)).max().item()


def _inputs(cfg: RunConfig, device):
    return tuple(gen_slots_device(cfg.seed, cfg.batch, cfg.heads, cfg.seq_len, cfg.dim, tag, dtype=cfg.dtype,
                                  device=device) for tag in ("q", "k", "v", "do"))


def _fd_eligible(cfg: RunConfig) -> bool:
    return cfg.precision == "f64" and cfg.seq_len <= _FD_MAX_N and cfg.dim <= _FD_MAX_D


def _grad_checks(cfg, tol_key, fn, arrays64, d64, got):
    tol = _TOLS[cfg.precision]
    ref = _grads(fn, arrays64, d64)
    checks = [Check("backward_rel_vs_oracle",
                    max(_error(g, r, cfg.precision, "rel") for g, r in zip(got, ref)), tol[tol_key])]
    if _fd_eligible(cfg):
        fd = _fd_grads(fn, arrays64, d64)
        checks.append(Check("backward_rel_vs_fd", max(_error(g, r, cfg.precision, "rel") for g, r in zip(got, fd)),
                            tol["fd"]))
    return checks


def _state_bytes(cfg: RunConfig) -> int:
    return cfg.batch * cfg.heads * cfg.dim * cfg.dim * costmodel.wire_element_bytes(cfg.element_bytes)


def _run_lasp2(cfg: RunConfig, corrupt: bool, device):
    q, k, v, do = _inputs(cfg, device)
    it = lasp2_iteration(ChunkedSequence(q, k, v, cfg.chunks), do, cfg.masked, cfg.world_config())
    out = _cat(it.outputs)
    got = [_cat(getattr(g, nm) for g in it.grads) for nm in ("dq", "dk", "dv")]
    if corrupt:
        got[0] = got[0] + 1e-3
    x64 = [x.double() for x in (q, k, v)]
    fn = lambda a, b, c: _linear_full(a, b, c, cfg.masked)  # noqa: E731
    tol = _TOLS[cfg.precision]
    checks = [Check("forward_max_abs_vs_oracle", _error(out, fn(*x64), cfg.precision, "abs"), tol["forward"])]
    checks += _grad_checks(cfg, "grad_serial", fn, x64, do.double(), got)
    st = it.run.stats
    dp = cfg.world // cfg.chunks
    checks.append(Check("collective_steps_exact", float(abs(st.allgather_launches - 2 * dp) + st.p2p_sends), 0.0))
    checks.append(Check("state_bytes_exact", float(abs(st.bytes_sent - 2 * cfg.world * _state_bytes(cfg))), 0.0))
    return checks, asdict(st), it.run.simulated_time


def _run_lasp1(cfg: RunConfig, corrupt: bool, device):
    q, k, v, do = _inputs(cfg, device)
    seq = ChunkedSequence(q, k, v, cfg.chunks)
    it = lasp1_iteration(seq, do, cfg.masked, cfg.world_config())
    out = _cat(it.outputs)
    got = [_cat(getattr(g, nm) for g in it.grads) for nm in ("dq", "dk", "dv")]
    if corrupt:
        got[0] = got[0] + 1e-3
    x64 = [x.double() for x in (q, k, v)]
    tol = _TOLS[cfg.precision]
    if cfg.masked:
        fn = lambda a, b, c: _linear_full(a, b, c, True)  # noqa: E731
        checks = [Check("forward_max_abs_vs_oracle", _error(out, fn(*x64), cfg.precision, "abs"), tol["forward"])]
        checks += _grad_checks(cfg, "grad_serial", fn, x64, do.double(), got)
        other = lasp2_iteration(seq, do, True, cfg.world_config())
        err = _error(out, _cat(other.outputs), cfg.precision, "rel")
        for mine, nm in zip(got, ("dq", "dk", "dv")):
            err = max(err, _error(mine, _cat(getattr(g, nm) for g in other.grads), cfg.precision, "rel"))
        checks.append(Check("vs_lasp2", err, tol["grad_serial"]))
    else:
        fn = lambda a, b, c: _exclusive_prefix_forward(a, b, c, cfg.chunks)  # noqa: E731
        checks = [Check("forward_vs_exclusive_prefix", _error(out, fn(*x64), cfg.precision, "abs"),
                        tol["forward"])]
        checks += [Check("backward_vs_exclusive_prefix", c.max_error, c.tolerance)
                   for c in _grad_checks(cfg, "grad_serial", fn, x64, do.double(), got)]
        ks, vs = (x.double().chunk(cfg.chunks, dim=2) for x in (k, v))
        full = sum(kc.transpose(-1, -2) @ vc for kc, vc in zip(ks, vs))
        checks.append(Check("ring_final_state", _error(it.caches[-1].state_through, full, cfg.precision, "rel"),
                            tol["grad_serial"]))
    st = it.run.stats
    dp = cfg.world // cfg.chunks
    checks.append(Check("ring_steps_exact",
                        float(abs(st.p2p_sends - dp * 2 * (cfg.chunks - 1)) + st.allgather_launches), 0.0))
    return checks, asdict(st), it.run.simulated_time


def _run_cp(cfg: RunConfig, corrupt: bool, device):
    q, k, v, do = _inputs(cfg, device)
    it = cp_iteration(ChunkedSequence(q, k, v, cfg.chunks), do, cfg.masked, cfg.world_config())
    out = _cat(it.outputs)
    got = [_cat(getattr(g, nm) for g in it.grads) for nm in ("dq", "dk", "dv")]
    if corrupt:
        got[0] = got[0] + 1e-3
    x64 = [x.double() for x in (q, k, v)]
    fn = lambda a, b, c: _softmax_full(a, b, c, cfg.masked)  # noqa: E731
    tol = _TOLS[cfg.precision]
    checks = [Check("forward_max_abs_vs_oracle", _error(out, fn(*x64), cfg.precision, "abs"),
                    tol["forward_softmax"])]
    checks += _grad_checks(cfg, "grad_softmax", fn, x64, do.double(), got)
    st = it.run.stats
    dp = cfg.world // cfg.chunks
    launches = st.allgather_launches + st.reduce_scatter_launches  # K, V gathers + the dK/dV reduce_scatter
    checks.append(Check("gather_launches_exact", float(abs(launches - 3 * dp) + st.p2p_sends), 0.0))
    chunk = cfg.seq_len // cfg.chunks
    per_rank = cfg.batch * cfg.heads * cfg.dim * (2 * chunk * cfg.element_bytes
                                                  + 2 * cfg.seq_len * costmodel.wire_element_bytes(cfg.element_bytes))
    checks.append(Check("gathered_bytes_exact", float(abs(st.bytes_sent - cfg.world * per_rank)), 0.0))
    return checks, asdict(st), it.run.simulated_time


def _stack_forward(layers, weights, x, causal):
    for kind, (wq, wk, wv) in zip(layers, weights):
        q, k, v = x @ wq, x @ wk, x @ wv
        x = _linear_full(q, k, v, causal) if kind == "L" else _softmax_full(q, k, v, causal)
    return x


def _run_lasp2h(cfg: RunConfig, corrupt: bool, device):
    spec = ModelSpec(pattern=cfg.pattern, dim=cfg.dim, heads=cfg.heads, batch=cfg.batch, seed=cfg.seed)
    x, dy = (gen_slots_device(cfg.seed, cfg.batch, cfg.heads, cfg.seq_len, cfg.dim, tag, dtype=cfg.dtype,
                              device=device) for tag in ("x", "do"))
    it = hybrid_iteration(spec, x, dy, cfg.chunks, cfg.masked, cfg.world_config())
    out, d_x = _cat(it.outputs), _cat(it.d_x)
    if corrupt:
        d_x = d_x + 1e-3
    layers = spec.layers
    # the weights as the run rounds them (bf16 / f32), evaluated in f64
    w64 = [tuple(torch.from_numpy(w).to(device).to(cfg.dtype).double() for w in ws) for ws in layer_weights(spec)]
    flat = [w for ws in w64 for w in ws]

    def fn(x_, *ws):
        return _stack_forward(layers, [ws[i:i + 3] for i in range(0, len(ws), 3)], x_, cfg.masked)

    ref = _grads(fn, [x.double(), *flat], dy.double())
    tol = _TOLS[cfg.precision]
    grad_err = _error(d_x, ref[0], cfg.precision, "rel")
    for got_w, ref_w in zip(it.d_weights, (ref[1 + i:4 + i] for i in range(0, len(flat), 3))):
        for g, r in zip(got_w, ref_w):
            grad_err = max(grad_err, _error(g, r, cfg.precision, "rel"))
    checks = [Check("forward_rel_vs_stack", _error(out, fn(x.double(), *flat), cfg.precision, "rel"), tol["stack"]),
              Check("backward_rel_vs_stack", grad_err, tol["stack"])]
    st = it.run.stats
    dp = cfg.world // cfg.chunks
    expected = (2 * layers.count("L") + 3 * layers.count("N")) * dp
    launches = st.allgather_launches + st.reduce_scatter_launches
    checks.append(Check("launch_composition_exact", float(abs(launches - expected) + st.p2p_sends), 0.0))
    return checks, asdict(st), it.run.simulated_time


_RUNNERS = {"lasp2": _run_lasp2, "lasp1": _run_lasp1, "cp": _run_cp, "lasp2h": _run_lasp2h}


def run_checks(cfg: RunConfig, corrupt: bool = False, device=None):
    """(checks, ledger dict, simulated_time) of one configuration."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    return _RUNNERS[cfg.method](cfg, corrupt, device)


def bench_row(cfg: RunConfig, device=None) -> list:
    """One BENCH_COLUMNS row: one iteration of the method (cli.py:695-726)."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    started = time.perf_counter_ns()
    if cfg.method == "lasp2h":
        spec = ModelSpec(pattern=cfg.pattern, dim=cfg.dim, heads=cfg.heads, batch=cfg.batch, seed=cfg.seed)
        x, dy = (gen_slots_device(cfg.seed, cfg.batch, cfg.heads, cfg.seq_len, cfg.dim, tag, dtype=cfg.dtype,
                                  device=device) for tag in ("x", "do"))
        run = hybrid_iteration(spec, x, dy, cfg.chunks, cfg.masked, cfg.world_config()).run
    else:
        q, k, v, do = _inputs(cfg, device)
        driver = {"lasp1": lasp1_iteration, "lasp2": lasp2_iteration, "cp": cp_iteration}[cfg.method]
        run = driver(ChunkedSequence(q, k, v, cfg.chunks), do, cfg.masked, cfg.world_config()).run
    torch.cuda.synchronize(device)
    wall = time.perf_counter_ns() - started
    st = run.stats
    return [cfg.method, cfg.seq_len, cfg.chunks, cfg.world, cfg.dim, cfg.heads, cfg.batch,
            "true" if cfg.masked else "false", st.communication_steps,
            st.allgather_launches + st.reduce_scatter_launches, st.bytes_sent, run.simulated_time, wall]


def cost_row(entry: dict) -> list:
    """One COST_COLUMNS row (cli.py:774-810); element_bytes defaults to 8 like the reference."""
    method = entry.get("method", "lasp2")
    world = entry.get("world", 1)
    try:
        p = costmodel.CostParams(world_size=world, sp_size=entry.get("chunks", world), batch=entry.get("batch", 1),
                                 heads=entry.get("heads", 1), dim=entry.get("dim", 8),
                                 iterations=entry.get("iterations", 1), element_bytes=entry.get("element_bytes", 8))
        return [method, p.world_size, p.sp_size, p.batch, p.heads, p.dim, p.element_bytes, p.iterations,
                costmodel.comm_steps_per_iteration(method, p.world_size), costmodel.traffic_per_step(p),
                costmodel.state_param_count(p.batch, p.heads, p.dim), costmodel.total_traffic(method, p)]
    except ValueError as exc:
        raise UsageError(str(exc)) from exc


_COST_DEFAULT_SHAPES = ((1, 1, 1, 4, 8, 1), (2, 1, 1, 4, 8, 1), (8, 2, 4, 8, 8, 1), (8, 2, 4, 8, 8, 10),
                        (64, 16, 16, 2048, 2, 1), (64, 16, 32, 4096, 2, 1))  # cli.py:751-758


def default_cost_grid() -> list[dict]:
    return [{"method": m, "world": w, "batch": b, "heads": h, "dim": d, "element_bytes": eb, "iterations": it}
            for m in costmodel.METHODS for (w, b, h, d, eb, it) in _COST_DEFAULT_SHAPES]


def default_verify_grid() -> list[dict]:
    """cli.py:623-637 without the 'oracle' method."""
    return [{"method": m, "seq_len": n, "chunks": t, "dim": d, "masked": masked,
             "pattern": "LN" if m == "lasp2h" else ""}
            for m in METHODS for n in (8, 64, 256) for t in (1, 2, 4, 8) if n % t == 0
            for d in (4, 16) for masked in (True, False)]


# ---- config files and flags (cli.py:552-620) --------------------------------------

_RUN_KEYS = ("method", "seq_len", "chunks", "world", "dim", "heads", "batch", "masked", "pattern", "precision",
             "seed", "latency_per_launch", "latency_per_byte")
_COST_KEYS = ("method", "world", "chunks", "batch", "heads", "dim", "element_bytes", "iterations")


def _entries(path: str, allowed) -> list[tuple[str, str, str]]:
    """(key as written, normalised key, raw value) of every 'key = value' line, comments
    and blank lines skipped, keys checked against `allowed` (cli.py:552-596)."""
    try:
        with open(path, encoding="utf-8") as fh:
            text = fh.read()
    except OSError as exc:
        raise UsageError(f"cannot read {path}: {exc}") from exc
    out = []
    for n, line in enumerate(text.splitlines(), 1):
        line = line.strip()
        if line and not line.startswith("#"):
            key, eq, value = (part.strip() for part in line.partition("="))
            if not eq:
                raise UsageError(f"{path}:{n}: expected key = value")
            name = key.strip().lstrip("-").replace("-", "_")
            if name not in _KEY_TYPES:
                raise UsageError(f"unknown configuration key {key!r}")
            if name not in allowed:
                raise UsageError(f"{path}: key {key!r} not valid here")
            out.append((key, name, value))
    return out


def _config_file(path: str, allowed) -> dict:
    return {name: _coerce(key, value)[1] for key, name, value in _entries(path, allowed)}


def _grid_file(path: str, allowed) -> list[dict]:
    """Cartesian product of comma-separated values, one axis per key."""
    axes: dict[str, list] = {}
    for key, name, value in _entries(path, allowed):
        if name in axes:
            raise UsageError(f"{path}: duplicate key {key!r}")
        axes[name] = [_coerce(key, piece.strip())[1] for piece in value.split(",")]
    if not axes:
        raise UsageError(f"{path}: grid file is empty")
    return [dict(zip(axes, combo)) for combo in itertools.product(*axes.values())]


def _expand(args, allowed, default_grid) -> list[dict]:
    base = _config_file(args.config, allowed) if args.config else {}
    for key in allowed:
        value = getattr(args, key, None)
        if value is not None:
            base[key] = _coerce(key, value)[1]
    if args.grid:
        return [dict(base, **entry) for entry in _grid_file(args.grid, allowed)]
    return [base] if base else default_grid()


def _write_csv(path: str | None, header: list[str], rows: list[list]) -> None:
    def emit(fh):
        writer = csv.writer(fh, lineterminator="\n")
        writer.writerow(header)
        writer.writerows(rows)

    if path:
        try:
            with open(path, "w", encoding="utf-8", newline="") as fh:
                emit(fh)
        except OSError as exc:
            raise UsageError(f"cannot write {path}: {exc}") from exc
    else:
        emit(sys.stdout)


def _describe(cfg: RunConfig) -> str:
    return (f"{cfg.method:<6} N={cfg.seq_len} T={cfg.chunks} W={cfg.world} d={cfg.dim} H={cfg.heads} "
            f"B={cfg.batch} masked={'true' if cfg.masked else 'false'} {cfg.precision} seed={cfg.seed}")


def cmd_verify(args) -> int:
    """cli.py:654-692: one line per run, a pass count, the JSON report with --out."""
    configs = [RunConfig(**d) for d in _expand(args, _RUN_KEYS, default_verify_grid)]
    records, failures = [], 0
    for cfg in configs:
        started = time.perf_counter_ns()
        checks, ledger, sim_time = run_checks(cfg, args.corrupt_gradient)
        wall = time.perf_counter_ns() - started
        passed = all(c.passed for c in checks)
        failures += 0 if passed else 1
        first = lambda prefix: next((c.max_error for c in checks if c.name.startswith(prefix)), None)  # noqa: E731
        records.append({"method": cfg.method, "config": asdict(cfg), "config_hash": cfg.config_hash(),
                        "seed": cfg.seed, "checks": [c.as_dict() for c in checks],
                        "forward_max_abs_error": first("forward"), "grad_max_rel_error": first("backward"),
                        "comm": ledger, "simulated_time": sim_time, "wall_time_ns": wall, "passed": passed})
        if passed:
            print(f"ok   {_describe(cfg)} checks={len(checks)}")
        else:
            worst = ", ".join(f"{c.name}={c.max_error:.3e}>{c.tolerance:g}" for c in checks if not c.passed)
            print(f"FAIL {_describe(cfg)} {worst}")
    print(f"{len(configs) - failures}/{len(configs)} runs passed")
    if args.out:
        try:
            with open(args.out, "w", encoding="utf-8") as fh:
                json.dump({"version": __version__, "runs": records}, fh, indent=2)
                fh.write("\n")
        except OSError as exc:
            raise UsageError(f"cannot write {args.out}: {exc}") from exc
    return 1 if failures else 0


def cmd_bench(args) -> int:
    configs = [RunConfig(**d) for d in _expand(args, _RUN_KEYS, lambda: [{}])]
    _write_csv(args.out, BENCH_COLUMNS, [bench_row(cfg) for cfg in configs])
    return 0


def cmd_costmodel(args) -> int:
    _write_csv(args.out, COST_COLUMNS, [cost_row(e) for e in _expand(args, _COST_KEYS, default_cost_grid)])
    return 0


def _run_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--method", choices=METHODS)
    p.add_argument("--seq-len", dest="seq_len", metavar="N")
    p.add_argument("--chunks", metavar="T")
    p.add_argument("--world", metavar="W")
    p.add_argument("--dim", metavar="D")
    p.add_argument("--heads", metavar="H")
    p.add_argument("--batch", metavar="B")
    p.add_argument("--masked", choices=["true", "false"])
    p.add_argument("--pattern", metavar="STR")
    p.add_argument("--precision", choices=sorted(PRECISIONS))
    p.add_argument("--seed", metavar="S")
    p.add_argument("--latency-per-launch", dest="latency_per_launch", metavar="COST")
    p.add_argument("--latency-per-byte", dest="latency_per_byte", metavar="COST")
    p.add_argument("--config", metavar="FILE")
    p.add_argument("--grid", metavar="FILE")
    p.add_argument("--out", metavar="PATH")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2502_07563_b200.harness",
                                     description="LASP-2 / LASP-2H on B200: verify, bench and cost tables.")
    parser.add_argument("--version", action="version", version=f"%(prog)s {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("verify", help="correctness checks; JSON report with --out")
    _run_flags(p)
    p.add_argument("--corrupt-gradient", dest="corrupt_gradient", action="store_true",
                   help="test hook: perturb a computed gradient so the failure path is exercised")
    p.set_defaults(func=cmd_verify)
    p = sub.add_parser("bench", help="one iteration per config; CSV to --out or stdout")
    _run_flags(p)
    p.set_defaults(func=cmd_bench)
    p = sub.add_parser("costmodel", help="closed-form step/traffic table; CSV to --out or stdout")
    for flag in ("method", "world", "chunks", "batch", "heads", "dim", "element-bytes", "iterations"):
        p.add_argument(f"--{flag}", dest=flag.replace("-", "_"),
                       **({"choices": costmodel.METHODS} if flag == "method" else {}))
    p.add_argument("--config", metavar="FILE")
    p.add_argument("--grid", metavar="FILE")
    p.add_argument("--out", metavar="PATH")
    p.set_defaults(func=cmd_costmodel)
    return parser


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return exc.code if isinstance(exc.code, int) else 2
    try:
        return args.func(args)
    except UsageError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
