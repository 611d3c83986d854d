"""Rank contexts for the LASP-2 hot path: the only collectives it needs.

Two implementations of one small interface (the subset of the reference's
RankContext that the hot path calls, comm.py:251-436):

* ``RankContext`` inside ``world_spawn`` — W ranks as host threads sharing one
  GPU, each with its own CUDA stream. It mirrors the reference simulator
  (threads-as-ranks, comm.py:465-531): payloads are snapshotted at hand-off,
  one collective launch per group per call, per-rank ledgers, a global trace,
  bounded waits that raise ``DeadlockError``. It lets every multi-rank parity
  test run on a single B200.
* ``DistRankContext`` — one process per GPU under torchrun; all_gather /
  reduce_scatter go to NCCL (``torch.distributed``) on a side stream so they
  overlap compute on the main stream; gloo works the same on CPU tensors.

Interface: ``sp_position``, ``sp_size``, ``all_gather_async(t) -> Pending``,
``all_gather(t)`` (returns the rank-ordered contributions stacked on a new
leading axis — the NCCL all_gather_into_tensor layout), ``reduce_scatter(t)``,
``send(dst, t)`` / ``recv(src)`` (the LASP-1 ring baseline's matched pairs;
NCCL P2P under torchrun), ``mark(kind)``, ``stats`` (CommStats) and ``trace``.
"""
from __future__ import annotations

import ctypes
import sys
import threading
import time
from collections import deque
from collections.abc import Callable, Sequence
from dataclasses import dataclass, field
from typing import Any

import torch


class CommError(Exception):
    """Base class for runtime communication failures (comm.py:31)."""


class DeadlockError(CommError):
    """A rank blocked past the configured timeout (comm.py:35)."""


class CollectiveError(CommError):
    """Participants disagreed about a collective's payload (comm.py:39)."""


class WorldAbortedError(CommError):
    """Another rank failed first (comm.py:43)."""


@dataclass(frozen=True)
class WorldConfig:
    """World layout (reference comm.py:51-87).

    world_size ranks form contiguous SP groups of sp_size; ranks at the same
    position across groups are DP peers. element_bytes is the data element
    size: 8 (f64), 4 (f32) or 2 (bf16, which exchanges f32 states). The
    latency fields drive the threads-as-ranks world's simulated clock
    (``WorldRun.simulated_time``, reference comm.py:7-12); real time is
    measured on the device (bench.py, ``WorldRun.device_timelines``).
    """

    world_size: int
    sp_size: int | None = None
    element_bytes: int = 8
    latency_per_launch: float = 10.0
    latency_per_byte: float = 1.0 / 1024.0
    deadlock_timeout: float = 120.0

    def __post_init__(self) -> None:
        if self.sp_size is None:
            object.__setattr__(self, "sp_size", self.world_size)
        if self.world_size < 1:
            raise ValueError(f"world_size must be >= 1, got {self.world_size}")
        if self.sp_size < 1:
            raise ValueError(f"sp_size must be >= 1, got {self.sp_size}")
        if self.world_size % self.sp_size != 0:
            raise ValueError(f"sp_size {self.sp_size} must divide world_size {self.world_size}")
        if self.element_bytes not in (2, 4, 8):
            raise ValueError(f"element_bytes must be 2, 4 or 8, got {self.element_bytes}")
        if self.deadlock_timeout <= 0:
            raise ValueError("deadlock_timeout must be positive")

    @property
    def dp_size(self) -> int:
        return self.world_size // self.sp_size


@dataclass
class CommStats:
    """Per-rank ledger (comm.py:90-105). One step = one collective launch."""

    p2p_sends: int = 0
    p2p_recvs: int = 0
    allgather_launches: int = 0
    reduce_scatter_launches: int = 0
    bytes_sent: int = 0
    communication_steps: int = 0
    bytes_by_primitive: dict[str, int] = field(default_factory=dict)

    def _account(self, primitive: str, nbytes: int) -> None:
        self.bytes_sent += nbytes
        self.bytes_by_primitive[primitive] = self.bytes_by_primitive.get(primitive, 0) + nbytes


@dataclass(frozen=True)
class TraceEvent:
    seq: int
    rank: int
    clock: float
    kind: str
    detail: str = ""


@dataclass(frozen=True)
class GroupInfo:
    dp_peers: tuple[int, ...]
    sp_peers: tuple[int, ...]
    sp_position: int


class PeerExchange:
    """One rank's handle on a fused peer-memory state exchange.

    ``recv`` [2, T, *state] is this rank's receive buffer, double-buffered by
    epoch parity (slot j = rank j's chunk total), ``flags`` [T] its
    epoch-stamped arrival flags, ``acks`` [T] the epochs each reader has
    finished folding (back-pressure for this rank's puts), ``*_table`` device
    arrays of every rank's buffer / flag / ack addresses (peer addresses over
    NVLink with symmetric memory; same-device addresses in the threads-as-ranks
    world), ``done`` the put kernel's completion counter, ``ep`` this rank's
    device-resident epoch (advanced by the put kernel itself, so a captured
    CUDA graph advances the exchange on every replay). ``ops.scan_put``
    writes, ``ops.exchange_fold`` waits, folds and acknowledges.
    """

    def __init__(self, rank: int, nranks: int, recv: torch.Tensor, flags: torch.Tensor, acks: torch.Tensor,
                 done: torch.Tensor, recv_table: torch.Tensor, flag_table: torch.Tensor,
                 ack_table: torch.Tensor) -> None:
        self.rank, self.nranks = rank, nranks
        self.recv, self.flags, self.acks, self.done = recv, flags, acks, done
        self.recv_table, self.flag_table, self.ack_table = recv_table, flag_table, ack_table
        self.ep = torch.zeros(1, dtype=torch.int64, device=recv.device)
        self.epoch = 0  # host count of exchanges issued (eager runs; a graph replay does not advance it)

    def next_epoch(self) -> int:
        self.epoch += 1
        return self.epoch


def _ptr_table(tensors: Sequence[torch.Tensor], device) -> torch.Tensor:
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64, device=device)


def process_groups(cfg: WorldConfig) -> dict[int, GroupInfo]:
    """Contiguous SP groups, strided DP peers (comm.py:143-158)."""
    t = cfg.sp_size
    out = {}
    for rank in range(cfg.world_size):
        g, pos = divmod(rank, t)
        out[rank] = GroupInfo(dp_peers=tuple(gg * t + pos for gg in range(cfg.dp_size)),
                              sp_peers=tuple(range(g * t, (g + 1) * t)), sp_position=pos)
    return out


class _ContextBase:
    """Shared trace / device-event bookkeeping."""

    rank: int
    stats: CommStats

    def _init_common(self) -> None:
        self.stats = CommStats()
        self.device_events: list[tuple[str, torch.cuda.Event]] = []

    def _device_mark(self, kind: str, stream=None) -> None:
        # timing events are for eager runs (bench.py's profiled pass); a captured graph
        # replays without them
        if torch.cuda.is_available() and torch.cuda.is_initialized() and \
                not torch.cuda.is_current_stream_capturing():
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream if stream is not None else torch.cuda.current_stream())
            self.device_events.append((kind, ev))

    def device_timeline(self) -> dict[str, list[float]]:
        """Milliseconds of every device mark relative to the first (call after a sync)."""
        if not self.device_events:
            return {}
        t0 = self.device_events[0][1]
        out: dict[str, list[float]] = {}
        for kind, ev in self.device_events:
            out.setdefault(kind, []).append(t0.elapsed_time(ev))
        return out


# ----------------------------------------------------------------------------
# Threads-as-ranks world on one GPU
# ----------------------------------------------------------------------------

class _Gen:
    __slots__ = ("shape", "dtype", "contributions", "complete", "error", "kind", "clocks", "completion_clock")

    def __init__(self, kind: str) -> None:
        self.kind = kind
        self.shape = None
        self.dtype = None
        self.contributions: dict[int, tuple[torch.Tensor, Any]] = {}
        self.complete = False
        self.error: CollectiveError | None = None
        self.clocks: dict[int, float] = {}  # simulated issue clock per rank
        self.completion_clock = 0.0


class _ClockGen:
    """Ledger-only generation of a collective (barriers, fused peer exchanges):
    issue clocks only, completion at the latest issue plus the transfer cost."""

    __slots__ = ("clocks", "completion_clock", "complete")

    def __init__(self) -> None:
        self.clocks: dict[int, float] = {}
        self.completion_clock = 0.0
        self.complete = False


class _World:
    def __init__(self, cfg: WorldConfig, device: torch.device) -> None:
        self.cfg = cfg
        self.device = device
        self.cond = threading.Condition(threading.Lock())
        self.trace: list[TraceEvent] = []
        self.abort_error: BaseException | None = None
        self.collective_launches = 0
        self.reduce_scatter_launches = 0
        t = cfg.sp_size
        self.groups = [tuple(range(g * t, (g + 1) * t)) for g in range(cfg.dp_size)]
        self.gens: dict[tuple[int, int], _Gen] = {}
        self.queues: dict[tuple[int, int], deque] = {}  # (src, dst) -> FIFO of (snapshot, event, sent clock)
        self.exchanges: dict[tuple, list[PeerExchange]] = {}  # (group, tag, shape, dtype) -> per-position handles
        self.clock_gens: dict[tuple, _ClockGen] = {}  # (group, kind, call) -> barrier / peer-exchange generation
        self.t0 = time.perf_counter()

    def record(self, rank: int, kind: str, detail: str) -> None:
        self.trace.append(TraceEvent(len(self.trace), rank, time.perf_counter() - self.t0, kind, detail))

    def abort(self, err: BaseException) -> None:
        if self.abort_error is None:
            self.abort_error = err
        self.cond.notify_all()

    def transfer_cost(self, nbytes: int) -> float:
        """Simulated cost of one step moving nbytes (reference comm.py:359-360, 403-404)."""
        return self.cfg.latency_per_launch + nbytes * self.cfg.latency_per_byte


class PendingGather:
    """Handle of an issued all_gather; wait() returns [T, *payload.shape]."""

    def __init__(self, ctx: "RankContext", key: tuple[int, int], tag: str) -> None:
        self._ctx = ctx
        self._key = key
        self._tag = tag
        self._result: torch.Tensor | None = None

    def wait(self) -> torch.Tensor:
        if self._result is not None:
            return self._result
        ctx = self._ctx
        world = ctx.world
        gen = world.gens[self._key]
        with world.cond:
            ctx._wait_locked(lambda: gen.complete or gen.error is not None,
                             lambda: f"all_gather call {self._key[1]} stalled: contributions from "
                                     f"{sorted(gen.contributions)}, group {ctx.sp_peers}")
            if gen.error is not None:
                raise CollectiveError(*gen.error.args)
            parts = [gen.contributions[r] for r in ctx.sp_peers]
            ctx.clock = max(ctx.clock, gen.completion_clock)
        stream = torch.cuda.current_stream()
        for _, ev in parts:
            stream.wait_event(ev)
        result = torch.stack([p for p, _ in parts])
        ctx._device_mark("all_gather_complete")
        with world.cond:
            world.record(ctx.rank, "all_gather_complete", f"call={self._key[1]} tag={self._tag}")
        self._result = result
        return result


class RankContext(_ContextBase):
    """One rank's handle inside ``world_spawn`` (reference comm.py:251-436)."""

    def __init__(self, world: _World, rank: int) -> None:
        self._init_common()
        self.world = world
        self.rank = rank
        self._group_index = rank // world.cfg.sp_size
        self._calls = 0
        self._barrier_calls = 0
        self.clock = 0.0  # simulated: only communication moves it (reference comm.py:7-12)
        self.stream = torch.cuda.Stream(device=world.device)

    @property
    def config(self) -> WorldConfig:
        return self.world.cfg

    @property
    def world_size(self) -> int:
        return self.world.cfg.world_size

    @property
    def sp_peers(self) -> tuple[int, ...]:
        return self.world.groups[self._group_index]

    @property
    def sp_position(self) -> int:
        return self.rank - self.sp_peers[0]

    @property
    def sp_size(self) -> int:
        return len(self.sp_peers)

    @property
    def dp_peers(self) -> tuple[int, ...]:
        t = self.world.cfg.sp_size
        return tuple(g * t + self.sp_position for g in range(self.world.cfg.dp_size))

    def _wait_locked(self, cond_fn: Callable[[], bool], describe: Callable[[], str]) -> None:
        deadline = time.monotonic() + self.world.cfg.deadlock_timeout
        while True:
            if self.world.abort_error is not None:
                raise WorldAbortedError(f"rank {self.rank}: aborted by {self.world.abort_error!r}")
            if cond_fn():
                return
            remaining = deadline - time.monotonic()
            if remaining <= 0:
                err = DeadlockError(f"rank {self.rank}: {describe()}")
                self.world.abort(err)
                raise err
            self.world.cond.wait(min(0.05, remaining))

    def _contribute(self, payload: torch.Tensor, tag: str, kind: str) -> tuple[tuple[int, int], int]:
        if not payload.is_cuda:
            raise ValueError("collective payloads must be CUDA tensors")
        snap = payload.detach().clone()  # frozen snapshot at hand-off (comm.py:299-302)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        nbytes = snap.numel() * snap.element_size()
        world = self.world
        with world.cond:
            if world.abort_error is not None:
                raise WorldAbortedError(f"rank {self.rank}: aborted by {world.abort_error!r}")
            call = self._calls
            self._calls += 1
            key = (self._group_index, call)
            gen = world.gens.setdefault(key, _Gen(kind))
            if gen.error is not None:
                raise CollectiveError(*gen.error.args)
            if gen.kind != kind:
                gen.error = CollectiveError(f"call {call}: rank {self.rank} issued {kind}, group issued {gen.kind}")
                world.cond.notify_all()
                raise gen.error
            if gen.shape is None:
                gen.shape, gen.dtype = tuple(snap.shape), snap.dtype
            elif tuple(snap.shape) != gen.shape or snap.dtype != gen.dtype:
                gen.error = CollectiveError(
                    f"{kind} call {call}: rank {self.rank} contributed {tuple(snap.shape)} {snap.dtype}, "
                    f"generation pinned to {gen.shape} {gen.dtype}")
                world.cond.notify_all()
                raise gen.error
            world.record(self.rank, f"{kind}_issue", f"call={call} tag={tag} bytes={nbytes}")
            gen.contributions[self.rank] = (snap, ev)
            gen.clocks[self.rank] = self.clock
            if len(gen.contributions) == len(self.sp_peers):
                gen.completion_clock = max(gen.clocks.values()) + world.transfer_cost(nbytes)
                gen.complete = True
                if kind == "all_gather":
                    world.collective_launches += 1
                else:
                    world.reduce_scatter_launches += 1
                world.cond.notify_all()
        self._device_mark(f"{kind}_issue")
        return key, nbytes

    def all_gather_async(self, payload: torch.Tensor, tag: str = "") -> PendingGather:
        key, nbytes = self._contribute(payload, tag, "all_gather")
        self.stats.allgather_launches += 1
        self.stats.communication_steps += 1
        self.stats._account("all_gather", nbytes)
        return PendingGather(self, key, tag)

    def all_gather(self, payload: torch.Tensor, tag: str = "") -> torch.Tensor:
        return self.all_gather_async(payload, tag).wait()

    def reduce_scatter(self, stacked: torch.Tensor, tag: str = "") -> torch.Tensor:
        """Sum of every rank's ``stacked[my_position]``, folded in ascending rank order."""
        if stacked.shape[0] != self.sp_size:
            raise ValueError(f"reduce_scatter expects a leading axis of {self.sp_size}, got {tuple(stacked.shape)}")
        key, nbytes = self._contribute(stacked, tag, "reduce_scatter")
        self.stats.reduce_scatter_launches += 1
        self.stats.communication_steps += 1
        self.stats._account("reduce_scatter", nbytes)
        world = self.world
        gen = world.gens[key]
        with world.cond:
            self._wait_locked(lambda: gen.complete or gen.error is not None,
                              lambda: f"reduce_scatter call {key[1]} stalled")
            if gen.error is not None:
                raise CollectiveError(*gen.error.args)
            parts = [gen.contributions[r] for r in self.sp_peers]
            self.clock = max(self.clock, gen.completion_clock)
        stream = torch.cuda.current_stream()
        for _, ev in parts:
            stream.wait_event(ev)
        pos = self.sp_position
        acc = parts[0][0][pos].clone()
        for p, _ in parts[1:]:
            acc += p[pos]
        self._device_mark("reduce_scatter_complete")
        return acc

    def reduce_to_owners(self, contrib: torch.Tensor, counts: Sequence[int], tag: str = "") -> torch.Tensor:
        """LASP-2H dK/dV exchange with per-rank contribution counts (rank t holds
        contributions to owners [0, counts[t])): in this world a zero-padded
        reduce_scatter, so ledger, bytes and simulated clock stay the reference's
        (standard_sp.py:69-75)."""
        t, pos = self.sp_size, self.sp_position
        if len(counts) != t or contrib.shape[0] != counts[pos]:
            raise ValueError(f"reduce_to_owners: contribution {tuple(contrib.shape)} does not match counts {counts}")
        padded = torch.zeros((t, *contrib.shape[1:]), dtype=contrib.dtype, device=contrib.device)
        padded[:counts[pos]] = contrib
        return self.reduce_scatter(padded, tag)

    def peer_exchange(self, tag: str, like: torch.Tensor) -> PeerExchange:
        """This rank's handle on the fused state exchange for states shaped like
        ``like`` (allocated once per group, tag, shape and dtype; every rank of
        the group shares the address tables)."""
        world = self.world
        key = (self._group_index, tag, tuple(like.shape), like.dtype)
        with world.cond:
            handles = world.exchanges.get(key)
            if handles is None:
                t, dev = self.sp_size, world.device
                recv = [torch.zeros((2, t, *like.shape), dtype=like.dtype, device=dev) for _ in range(t)]
                flags = [torch.zeros(t, dtype=torch.int64, device=dev) for _ in range(t)]
                acks = [torch.zeros(t, dtype=torch.int64, device=dev) for _ in range(t)]
                done = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(t)]
                tables = [_ptr_table(x, dev) for x in (recv, flags, acks)]
                torch.cuda.synchronize(dev)  # zero-filled before any rank's kernels touch them
                handles = [PeerExchange(p, t, recv[p], flags[p], acks[p], done[p], *tables) for p in range(t)]
                world.exchanges[key] = handles
        return handles[self.sp_position]

    def _clock_collective(self, kind: str, call: int, nbytes: int | None, on_complete=None) -> None:
        """Join ledger-only generation (group, kind, call) and advance this rank's
        simulated clock to its completion: the latest issue plus, when nbytes is
        given, one transfer (a barrier aligns clocks at no cost, comm.py:414-431).
        Called with world.cond held."""
        world = self.world
        gen = world.clock_gens.setdefault((self._group_index, kind, call), _ClockGen())
        gen.clocks[self.rank] = self.clock
        if len(gen.clocks) == self.sp_size:
            latest = max(gen.clocks.values())
            gen.completion_clock = latest if nbytes is None else latest + world.transfer_cost(nbytes)
            gen.complete = True
            if on_complete is not None:
                on_complete()
            world.cond.notify_all()
        self._wait_locked(lambda: gen.complete, lambda: f"{kind} call {call} stalled: arrived {sorted(gen.clocks)}")
        self.clock = max(self.clock, gen.completion_clock)

    def account_exchange(self, ex: PeerExchange, tag: str = "") -> None:
        """Ledger of one fused exchange: one all_gather launch per group per call,
        this rank's contribution in bytes (comm.py:395-397); the simulated clock
        advances as for a blocking all_gather (the consumers' in-kernel waits
        are the device-side join)."""
        nbytes = ex.recv[0, 0].numel() * ex.recv.element_size()
        world = self.world
        with world.cond:
            call = self._calls
            self._calls += 1
            world.record(self.rank, "all_gather_issue", f"call={call} tag={tag} bytes={nbytes} peer")

            def launched() -> None:
                world.collective_launches += 1

            self._clock_collective("peer_exchange", call, nbytes, launched)
        self.stats.allgather_launches += 1
        self.stats.communication_steps += 1
        self.stats._account("all_gather", nbytes)
        self._device_mark("all_gather_issue")

    def send(self, dst: int, payload: torch.Tensor, tag: str = "") -> None:
        """Deposit a frozen snapshot for global rank dst; non-blocking. The
        matched pair is one communication step on the sender's ledger (comm.py:324-343)."""
        if not 0 <= dst < self.world_size:
            raise ValueError(f"destination {dst} outside world of {self.world_size}")
        if not payload.is_cuda:
            raise ValueError("p2p payloads must be CUDA tensors")
        snap = payload.detach().clone()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        nbytes = snap.numel() * snap.element_size()
        world = self.world
        with world.cond:
            if world.abort_error is not None:
                raise WorldAbortedError(f"rank {self.rank}: aborted by {world.abort_error!r}")
            world.record(self.rank, "send", f"dst={dst} tag={tag} bytes={nbytes}")
            self.stats.p2p_sends += 1
            self.stats.communication_steps += 1
            self.stats._account("send", nbytes)
            world.queues.setdefault((self.rank, dst), deque()).append((snap, ev, self.clock))
            world.cond.notify_all()
        self._device_mark("send")

    def recv(self, src: int, tag: str = "") -> torch.Tensor:
        """Next message from global rank src (FIFO per channel; the tag labels,
        it does not filter), ordered after the sender's stream (comm.py:345-365)."""
        if not 0 <= src < self.world_size:
            raise ValueError(f"source {src} outside world of {self.world_size}")
        if src == self.rank:
            raise ValueError(f"rank {self.rank} cannot receive from itself")
        world = self.world
        with world.cond:
            queue = world.queues.setdefault((src, self.rank), deque())
            self._wait_locked(lambda: len(queue) > 0, lambda: f"recv from rank {src} found no matching send")
            snap, ev, sent_clock = queue.popleft()
            nbytes = snap.numel() * snap.element_size()
            self.clock = max(self.clock, sent_clock + world.transfer_cost(nbytes))
            self.stats.p2p_recvs += 1
            world.record(self.rank, "recv", f"src={src} tag={tag} bytes={nbytes}")
        torch.cuda.current_stream().wait_event(ev)
        self._device_mark("recv")
        return snap

    def barrier(self) -> None:
        """Synchronise the SP group host-side: clocks align, no bytes or steps
        accrue (comm.py:414-431). Device order is the callers' business."""
        world = self.world
        with world.cond:
            call = self._barrier_calls
            self._barrier_calls += 1
            world.record(self.rank, "barrier", f"call={call}")
            self._clock_collective("barrier", call, None)

    def mark(self, kind: str, detail: str = "") -> None:
        with self.world.cond:
            self.world.record(self.rank, kind, detail)
        self._device_mark(kind)


@dataclass
class WorldRun:
    """Everything a completed world leaves behind (comm.py:439-448)."""

    config: WorldConfig
    results: list[Any]
    rank_stats: list[CommStats]
    stats: CommStats
    trace: list[TraceEvent]
    device_timelines: list[dict[str, list[float]]]
    wall_seconds: float
    simulated_time: float | None = None  # threads-as-ranks world only: max final rank clock (comm.py:530)


def _merge_stats(rank_stats: Sequence[CommStats], ag_launches: int, rs_launches: int) -> CommStats:
    merged = CommStats()
    for st in rank_stats:
        merged.p2p_sends += st.p2p_sends
        merged.p2p_recvs += st.p2p_recvs
        merged.bytes_sent += st.bytes_sent
        for key, val in st.bytes_by_primitive.items():
            merged.bytes_by_primitive[key] = merged.bytes_by_primitive.get(key, 0) + val
    merged.allgather_launches = ag_launches
    merged.reduce_scatter_launches = rs_launches
    merged.communication_steps = merged.p2p_sends + ag_launches + rs_launches
    return merged


def world_spawn(cfg: WorldConfig, program: Callable[..., Any], rank_args: Sequence[tuple] | None = None,
                device: torch.device | None = None) -> WorldRun:
    """Run program(ctx, *rank_args[rank]) on one host thread per rank, all on one GPU (comm.py:465-531)."""
    if rank_args is not None and len(rank_args) != cfg.world_size:
        raise ValueError(f"rank_args has {len(rank_args)} entries for {cfg.world_size} ranks")
    if not torch.cuda.is_available():
        raise RuntimeError("world_spawn needs a CUDA device (the LASP-2 B200 path has no CPU fallback)")
    device = device or torch.device("cuda", torch.cuda.current_device())
    world = _World(cfg, device)
    ctxs = [RankContext(world, r) for r in range(cfg.world_size)]
    results: list[Any] = [None] * cfg.world_size
    errors: list[BaseException | None] = [None] * cfg.world_size
    launcher = torch.cuda.current_stream(device)
    for ctx in ctxs:
        ctx.stream.wait_stream(launcher)

    def runner(ctx: RankContext) -> None:
        args = rank_args[ctx.rank] if rank_args is not None else ()
        try:
            torch.cuda.set_device(device)
            with torch.cuda.stream(ctx.stream):
                ctx._device_mark("start")
                results[ctx.rank] = program(ctx, *args)
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            errors[ctx.rank] = exc
            with world.cond:
                world.abort(exc)

    t0 = time.perf_counter()
    threads = [threading.Thread(target=runner, args=(c,), name=f"rank{c.rank}") for c in ctxs]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    torch.cuda.synchronize(device)
    wall = time.perf_counter() - t0
    for ctx in ctxs:
        launcher.wait_stream(ctx.stream)

    primary = next((e for e in errors if e is not None and not isinstance(e, WorldAbortedError)), None)
    if primary is None:
        primary = next((e for e in errors if e is not None), None)
    if primary is not None:
        raise primary
    return WorldRun(config=cfg, results=results, rank_stats=[c.stats for c in ctxs],
                    stats=_merge_stats([c.stats for c in ctxs], world.collective_launches,
                                       world.reduce_scatter_launches),
                    trace=list(world.trace), device_timelines=[c.device_timeline() for c in ctxs],
                    wall_seconds=wall, simulated_time=max(c.clock for c in ctxs))


# ----------------------------------------------------------------------------
# One process per GPU (torchrun): NCCL on a side stream, gloo on CPU
# ----------------------------------------------------------------------------

class DistPending:
    def __init__(self, ctx: "DistRankContext", work, out: torch.Tensor, tag: str) -> None:
        self._ctx = ctx
        self._work = work
        self._out = out
        self._tag = tag
        self._done = False

    def wait(self) -> torch.Tensor:
        if not self._done:
            ctx = self._ctx
            if self._out.is_cuda:
                with torch.cuda.stream(ctx.comm_stream):
                    self._work.wait()
                    ctx._device_mark("all_gather_complete", ctx.comm_stream)
                torch.cuda.current_stream().wait_stream(ctx.comm_stream)
                if not torch.cuda.is_current_stream_capturing():
                    self._out.record_stream(torch.cuda.current_stream())
            else:
                self._work.wait()
            ctx.trace.append(TraceEvent(len(ctx.trace), ctx.rank, time.perf_counter(), "all_gather_complete",
                                        f"tag={self._tag}"))
            self._done = True
        return self._out


class NcclComm:
    """An NCCL communicator driven through the C ABI's collective wrappers
    (lasp2_state_allgather, lasp2h_kv_allgather, lasp2h_grad_reduce_scatter;
    SURVEY §8b). Every call is enqueued on the given (default: current) stream."""

    def __init__(self, nranks: int, rank: int, unique_id: bytes) -> None:
        from . import _lib

        if len(unique_id) != 128:
            raise ValueError("an NCCL unique id is 128 bytes")
        self._lib = _lib
        self.nranks, self.rank = nranks, rank
        handle = ctypes.c_void_p()
        uid = ctypes.create_string_buffer(bytes(unique_id), 128)
        _lib.call("lasp2_nccl_comm_init", ctypes.addressof(handle), nranks, ctypes.addressof(uid), rank)
        self.handle = handle.value

    @staticmethod
    def unique_id() -> bytes:
        from . import _lib

        buf = ctypes.create_string_buffer(128)
        _lib.call("lasp2_nccl_unique_id", ctypes.addressof(buf))
        return buf.raw

    def _stream(self, stream) -> int:
        return self._lib.stream_ptr(stream)

    def all_gather(self, payload: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """[nranks, *payload.shape], rank-major (the state AllGather)."""
        payload = payload.contiguous()
        if out is None:
            out = torch.empty((self.nranks, *payload.shape), dtype=payload.dtype, device=payload.device)
        self._lib.call("lasp2_state_allgather", self.handle, self._lib.dtype_code(payload.dtype), payload.data_ptr(),
                       out.data_ptr(), payload.numel(), self._stream(stream))
        return out

    def all_gather_kv(self, k: torch.Tensor, v: torch.Tensor, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
        """LASP-2H K and V gathers (two launches), each [nranks, *chunk.shape]."""
        k, v = k.contiguous(), v.contiguous()
        kf = torch.empty((self.nranks, *k.shape), dtype=k.dtype, device=k.device)
        vf = torch.empty_like(kf)
        self._lib.call("lasp2h_kv_allgather", self.handle, self._lib.dtype_code(k.dtype), k.data_ptr(), v.data_ptr(),
                       kf.data_ptr(), vf.data_ptr(), k.numel(), self._stream(stream))
        return kf, vf

    def reduce_scatter(self, stacked: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Sum over ranks of stacked[my rank] (stacked: [nranks, ...])."""
        if stacked.shape[0] != self.nranks:
            raise ValueError(f"reduce_scatter expects a leading axis of {self.nranks}, got {tuple(stacked.shape)}")
        stacked = stacked.contiguous()
        if out is None:
            out = torch.empty(stacked.shape[1:], dtype=stacked.dtype, device=stacked.device)
        self._lib.call("lasp2h_grad_reduce_scatter", self.handle, self._lib.dtype_code(stacked.dtype),
                       stacked.data_ptr(), out.data_ptr(), out.numel(), self._stream(stream))
        return out

    def close(self) -> None:
        if self.handle:
            self._lib.call("lasp2_nccl_comm_destroy", self.handle)
            self.handle = None


class _Done:
    def wait(self) -> None:
        return None


class DistRankContext(_ContextBase):
    """Rank context over an initialised torch.distributed default group.

    SP groups are contiguous blocks of ``sp_size`` ranks (comm.py:143-158);
    every process must construct its context (new_group is collective).
    """

    one_gpu_per_rank = True  # consumers may wait for peers inside their kernels

    def __init__(self, sp_size: int | None = None, peer_exchange: bool = False,
                 native_collectives: bool = False) -> None:
        import torch.distributed as dist

        self._init_common()
        self._peer = peer_exchange
        self.peer_fallback: str | None = None  # why a requested peer exchange is not in use
        self.peer_method: str | None = None    # "symmetric_memory" or "cuda_ipc" once rendezvoused
        self._exchanges: dict[tuple, PeerExchange] = {}
        self.dist = dist
        self.rank = dist.get_rank()
        world = dist.get_world_size()
        sp = sp_size or world
        if world % sp:
            raise ValueError(f"sp_size {sp} must divide world size {world}")
        self._sp_size = sp
        self._group = None
        if sp == world:
            self._group = dist.group.WORLD
        else:
            for g in range(world // sp):
                ranks = list(range(g * sp, (g + 1) * sp))
                pg = dist.new_group(ranks)
                if self.rank in ranks:
                    self._group = pg
        self.trace: list[TraceEvent] = []
        self.comm_stream = torch.cuda.Stream() if torch.cuda.is_available() else None
        # gloo moves host memory: device payloads are staged through the host (synchronous;
        # the multi-process tests run several ranks on one GPU this way, NCCL refuses that)
        self._stage = dist.get_backend(self._group) == "gloo"
        # native_collectives: the state / K,V gathers and the dK,dV reduce-scatter go through
        # the C ABI's NCCL wrappers on this context's own communicator (one per SP group)
        self.nccl: NcclComm | None = None
        if native_collectives:
            leader = self.rank - self.rank % sp
            uid = [NcclComm.unique_id() if self.rank == leader else None]
            dist.broadcast_object_list(uid, src=leader, group=self._group)
            self.nccl = NcclComm(sp, self.rank % sp, uid[0])

    @property
    def sp_position(self) -> int:
        return self.rank % self._sp_size

    @property
    def sp_size(self) -> int:
        return self._sp_size

    def _account(self, kind: str, t: torch.Tensor) -> None:
        nbytes = t.numel() * t.element_size()
        if kind == "all_gather":
            self.stats.allgather_launches += 1
        else:
            self.stats.reduce_scatter_launches += 1
        self.stats.communication_steps += 1
        self.stats._account(kind, nbytes)
        self.trace.append(TraceEvent(len(self.trace), self.rank, time.perf_counter(), f"{kind}_issue",
                                     f"bytes={nbytes}"))

    def all_gather_async(self, payload: torch.Tensor, tag: str = "") -> DistPending:
        payload = payload.contiguous()
        if payload.ndim == 0:
            payload = payload.reshape(1)
        # gathered along dim 0 (the layout gloo and NCCL both accept), viewed [T, *payload.shape]
        flat = torch.empty((self._sp_size * payload.shape[0], *payload.shape[1:]), dtype=payload.dtype,
                           device=payload.device)
        out = flat.view(self._sp_size, *payload.shape)
        self._account("all_gather", payload)
        if payload.is_cuda and self._stage:
            host = torch.empty(flat.shape, dtype=flat.dtype)
            self.dist.all_gather_into_tensor(host, payload.cpu(), group=self._group)
            flat.copy_(host)
            work = _Done()
        elif payload.is_cuda:
            cur = torch.cuda.current_stream()
            self.comm_stream.wait_stream(cur)
            with torch.cuda.stream(self.comm_stream):
                self._device_mark("all_gather_issue", self.comm_stream)
                if self.nccl is not None:
                    self.nccl.all_gather(payload, out=out, stream=self.comm_stream)
                    work = _Done()
                else:
                    work = self.dist.all_gather_into_tensor(flat, payload, group=self._group, async_op=True)
            if not torch.cuda.is_current_stream_capturing():
                payload.record_stream(self.comm_stream)
                flat.record_stream(self.comm_stream)
        else:
            work = self.dist.all_gather_into_tensor(flat, payload, group=self._group, async_op=True)
        return DistPending(self, work, out, tag)

    def all_gather(self, payload: torch.Tensor, tag: str = "") -> torch.Tensor:
        return self.all_gather_async(payload, tag).wait()

    def reduce_scatter(self, stacked: torch.Tensor, tag: str = "") -> torch.Tensor:
        if stacked.shape[0] != self._sp_size:
            raise ValueError(f"reduce_scatter expects a leading axis of {self._sp_size}, got {tuple(stacked.shape)}")
        stacked = stacked.contiguous()
        out = torch.empty(stacked.shape[1:], dtype=stacked.dtype, device=stacked.device)
        self._account("reduce_scatter", stacked)
        if self.nccl is not None and stacked.is_cuda:
            return self.nccl.reduce_scatter(stacked, out=out)
        if stacked.is_cuda and self._stage:
            host = torch.empty(out.shape, dtype=out.dtype)
            self.dist.reduce_scatter_tensor(host.view(-1), stacked.view(-1).cpu(), group=self._group)
            return out.copy_(host)
        flat_in = stacked.view(-1)
        self.dist.reduce_scatter_tensor(out.view(-1), flat_in, group=self._group)
        return out

    def reduce_to_owners(self, contrib: torch.Tensor, counts: Sequence[int], tag: str = "") -> torch.Tensor:
        """The LASP-2H dK/dV reduction without the causal zeros: rank t holds contributions
        to owners (key chunks) [0, counts[t]); owner r receives them from every rank with
        counts[t] > r over point-to-point transfers (one NCCL group) and folds them in
        ascending rank order, copy-first, as the reference's sum over ranks
        (standard_sp.py:69-75). With contiguous causal chunks counts[t] = t + 1, so a rank
        sends t chunks instead of the reduce_scatter's T - 1. Ledger: one reduce_scatter
        launch with the bytes this rank actually sends."""
        t_world, pos = self._sp_size, self.sp_position
        if len(counts) != t_world or contrib.shape[0] != counts[pos]:
            raise ValueError(f"reduce_to_owners: contribution {tuple(contrib.shape)} does not match counts {counts}")
        contrib = contrib.contiguous()
        peers = self.sp_peers
        senders = [r for r in range(t_world) if r != pos and counts[r] > pos]
        targets = [r for r in range(counts[pos]) if r != pos]
        esize = contrib[0].numel() * contrib.element_size()
        nbytes = esize * len(targets)
        self.stats.reduce_scatter_launches += 1
        self.stats.communication_steps += 1
        self.stats._account("reduce_scatter", nbytes)
        self.trace.append(TraceEvent(len(self.trace), self.rank, time.perf_counter(), "reduce_scatter_issue",
                                     f"bytes={nbytes} owners tag={tag}"))
        stage = self._stage and contrib.is_cuda
        src = contrib.cpu() if stage else contrib
        recv = {r: torch.empty(contrib.shape[1:], dtype=contrib.dtype, device=src.device) for r in senders}
        ops = [self.dist.P2POp(self.dist.irecv, recv[r], peers[r]) for r in senders]
        ops += [self.dist.P2POp(self.dist.isend, src[r], peers[r]) for r in targets]
        if ops:
            for work in self.dist.batch_isend_irecv(ops):
                work.wait()
        acc = None
        for r in range(t_world):
            if r == pos and pos < counts[pos]:
                part = contrib[pos]
            elif r in recv:
                part = recv[r].to(contrib.device, non_blocking=True) if stage else recv[r]
            else:
                continue
            if acc is None:
                acc = part.clone()
            else:
                acc += part
        if acc is None:
            acc = torch.zeros(contrib.shape[1:], dtype=contrib.dtype, device=contrib.device)
        return acc

    @property
    def sp_peers(self) -> tuple[int, ...]:
        g = self.rank // self._sp_size
        return tuple(range(g * self._sp_size, (g + 1) * self._sp_size))

    def peer_exchange(self, tag: str, like: torch.Tensor) -> PeerExchange | None:
        """Fused state exchange over NVLink peer memory (torch symmetric memory),
        opted in with ``DistRankContext(peer_exchange=True)``; None keeps the
        NCCL all_gather. Buffers are allocated once per (tag, shape, dtype)."""
        if not self._peer or not like.is_cuda:
            return None
        key = (tag, tuple(like.shape), like.dtype)
        ex = self._exchanges.get(key)
        if ex is None:
            errors = []
            for method in ("symmetric_memory", "cuda_ipc"):
                err = None
                try:
                    ex = (self._rendezvous_exchange if method == "symmetric_memory" else
                          self._rendezvous_exchange_ipc)(like)
                except Exception as exc:  # noqa: BLE001 - reported, then the next method runs
                    err, ex = f"{method}: {type(exc).__name__}: {exc}", None
                # the group agrees (MIN over ranks) so that all ranks keep one exchange protocol
                ok = torch.tensor([0 if err else 1], dtype=torch.int32,
                                  device="cpu" if self._stage else like.device)  # gloo reduces host tensors
                self.dist.all_reduce(ok, op=self.dist.ReduceOp.MIN, group=self._group)
                if int(ok.item()):
                    self.peer_method = method
                    break
                errors.append(err or f"{method}: another rank of the group failed the rendezvous")
                ex = None
            if ex is None:
                self._peer = False
                self.peer_fallback = "; ".join(errors)
                print(f"[lasp2] rank {self.rank}: peer state exchange unavailable ({self.peer_fallback}); "
                      f"falling back to the NCCL all_gather", file=sys.stderr, flush=True)
                return None
            if errors:
                print(f"[lasp2] rank {self.rank}: peer state exchange over {self.peer_method} "
                      f"({'; '.join(errors)})", file=sys.stderr, flush=True)
            self._exchanges[key] = ex
        return ex

    def _rendezvous_exchange_ipc(self, like: torch.Tensor) -> PeerExchange:
        """The same buffers mapped into every rank of the group with CUDA IPC handles
        (torch's own tensor-sharing reductions, exchanged with all_gather_object): works
        where symmetric memory refuses, e.g. several ranks on one device, and for peer
        devices with P2P access (the mapping enables it lazily)."""
        from torch.multiprocessing.reductions import reduce_tensor

        t, dev = self._sp_size, like.device
        bufs = [torch.zeros((2, t, *like.shape), dtype=like.dtype, device=dev),
                torch.zeros((t,), dtype=torch.int64, device=dev),
                torch.zeros((t,), dtype=torch.int64, device=dev)]
        torch.cuda.synchronize(dev)
        mine = [reduce_tensor(b) for b in bufs]
        everyone: list = [None] * t
        self.dist.all_gather_object(everyone, mine, group=self._group)
        self._ipc_keep = getattr(self, "_ipc_keep", [])  # peers' mappings live as long as the context
        tables = []
        for i, buf in enumerate(bufs):
            ptrs = []
            for r in range(t):
                if r == self.sp_position:
                    ptrs.append(buf.data_ptr())
                else:
                    fn, args = everyone[r][i]
                    peer = fn(*args)
                    self._ipc_keep.append(peer)
                    ptrs.append(peer.data_ptr())
            tables.append(torch.tensor(ptrs, dtype=torch.int64, device=dev))
        self._ipc_keep.extend(bufs)
        torch.cuda.synchronize(dev)
        self.dist.barrier(group=self._group)  # every rank's zero-fill and mapping precede any put
        return PeerExchange(self.sp_position, t, *bufs, torch.zeros(1, dtype=torch.int32, device=dev), *tables)

    def _rendezvous_exchange(self, like: torch.Tensor) -> PeerExchange:
        import torch.distributed._symmetric_memory as symm_mem

        t, dev = self._sp_size, like.device
        group_name = self._group.group_name
        bufs = [symm_mem.empty((2, t, *like.shape), dtype=like.dtype, device=dev),
                symm_mem.empty((t,), dtype=torch.int64, device=dev),
                symm_mem.empty((t,), dtype=torch.int64, device=dev)]
        tables = []
        for buf in bufs:
            buf.zero_()
            hdl = symm_mem.rendezvous(buf, group_name)
            if hdl.buffer_ptrs[hdl.rank] != buf.data_ptr():
                raise RuntimeError("symmetric-memory buffer is not at the start of its allocation")
            tables.append(torch.tensor(list(hdl.buffer_ptrs), dtype=torch.int64, device=dev))
        torch.cuda.synchronize(dev)
        self.dist.barrier(group=self._group)  # every rank's zero-fill precedes any put
        return PeerExchange(self.sp_position, t, *bufs, torch.zeros(1, dtype=torch.int32, device=dev), *tables)

    def account_exchange(self, ex: PeerExchange, tag: str = "") -> None:
        nbytes = ex.recv[0, 0].numel() * ex.recv.element_size()
        self.stats.allgather_launches += 1
        self.stats.communication_steps += 1
        self.stats._account("all_gather", nbytes)
        self.trace.append(TraceEvent(len(self.trace), self.rank, time.perf_counter(), "all_gather_issue",
                                     f"bytes={nbytes} peer tag={tag}"))

    def send(self, dst: int, payload: torch.Tensor, tag: str = "") -> None:
        """Point-to-point send to global rank dst (NCCL P2P over NVLink / gloo on CPU)."""
        payload = payload.contiguous()
        nbytes = payload.numel() * payload.element_size()
        self.stats.p2p_sends += 1
        self.stats.communication_steps += 1
        self.stats._account("send", nbytes)
        self.trace.append(TraceEvent(len(self.trace), self.rank, time.perf_counter(), "send",
                                     f"dst={dst} tag={tag} bytes={nbytes}"))
        self.dist.send(payload.cpu() if payload.is_cuda and self._stage else payload, dst)

    def recv(self, src: int, tag: str = "", like: torch.Tensor | None = None) -> torch.Tensor:
        """Receive into a fresh tensor shaped like ``like`` (the ring's payloads
        have the sender's shape and dtype, known to the receiver)."""
        if like is None:
            raise ValueError("DistRankContext.recv needs a template tensor (like=)")
        out = torch.empty_like(like)
        if out.is_cuda and self._stage:
            host = torch.empty(out.shape, dtype=out.dtype)
            self.dist.recv(host, src)
            out.copy_(host)
        else:
            self.dist.recv(out, src)
        self.stats.p2p_recvs += 1
        self.trace.append(TraceEvent(len(self.trace), self.rank, time.perf_counter(), "recv", f"src={src} tag={tag}"))
        return out

    def barrier(self) -> None:
        self.dist.barrier(group=self._group)

    def mark(self, kind: str, detail: str = "") -> None:
        self.trace.append(TraceEvent(len(self.trace), self.rank, time.perf_counter(), kind, detail))
        self._device_mark(kind)


class LocalRankContext(_ContextBase):
    """World of one rank (T = 1) without torch.distributed: collectives are
    local, still accounted as one launch each (the bench's N=1 path)."""

    def __init__(self) -> None:
        self._init_common()
        self.rank = 0
        self.trace: list[TraceEvent] = []

    sp_position = 0
    sp_size = 1

    def _account(self, kind: str, t: torch.Tensor) -> None:
        if kind == "all_gather":
            self.stats.allgather_launches += 1
        else:
            self.stats.reduce_scatter_launches += 1
        self.stats.communication_steps += 1
        self.stats._account(kind, t.numel() * t.element_size())

    def all_gather_async(self, payload: torch.Tensor, tag: str = ""):
        self._account("all_gather", payload)
        out = payload.unsqueeze(0)

        class _Done:
            def wait(self_inner):
                return out

        return _Done()

    def all_gather(self, payload: torch.Tensor, tag: str = "") -> torch.Tensor:
        return self.all_gather_async(payload, tag).wait()

    def reduce_scatter(self, stacked: torch.Tensor, tag: str = "") -> torch.Tensor:
        self._account("reduce_scatter", stacked)
        return stacked[0]

    def reduce_to_owners(self, contrib: torch.Tensor, counts: Sequence[int], tag: str = "") -> torch.Tensor:
        return self.reduce_scatter(contrib[:1], tag)

    sp_peers = (0,)

    def peer_exchange(self, tag: str, like: torch.Tensor) -> None:
        return None  # a world of one exchanges nothing (the all_gather is the identity)

    def send(self, dst: int, payload: torch.Tensor, tag: str = "") -> None:
        raise ValueError(f"destination {dst} outside world of 1")

    def recv(self, src: int, tag: str = "", like: torch.Tensor | None = None) -> torch.Tensor:
        raise ValueError(f"source {src} outside world of 1")

    def barrier(self) -> None:
        pass

    def mark(self, kind: str, detail: str = "") -> None:
        pass
