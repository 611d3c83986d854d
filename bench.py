"""LASP-2 layer benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Headline workload (BASELINE.json configs[1], the first GPU config):
cfg2 = LASP-2 unmasked (bidirectional) layer fwd+bwd, B=1 H=16 d=128,
N=131072 tokens in total, C = N/W per GPU (strong scaling, as the config fixes N).
The same line carries the masked cfg3 layer (N=524288, the Linear-Llama3-1B
shape) under "secondary", measured the same way.

One step = rank_forward + rank_backward of one layer on the rank's chunk
(state all_gather over NCCL for N>1). Inputs (SplitMix64 counter-hash, the
reference datagen, generated on device) are 2 GiB+ per step, far above the
126 MB L2, so no flush is needed. Device time = CUDA events on the compute
stream between barrier+synchronize brackets, max over ranks.

--impl reference times the reference algorithm's CPU implementation (the
numpy oracle port under oracle/, f32, all host cores) on the same config: cfg2
at its full N with T = --gpus chunks (same `config` object as this arm), the
masked / LASP-2H workloads at the largest N the port runs in seconds
(labelled, never extrapolated); rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LASP-2 fwd+bwd tokens/sec at 1/2/4/8 B200, % of bf16 tensor peak"
UNIT = "tokens/s"
H, D, B = 16, 128, 1
WORKLOADS = {
    "cfg2": dict(name="cfg2: LASP-2 unmasked (bidirectional) layer fwd+bwd, B=1 H=16 d=128, N=131072 total",
                 n=131072, masked=False),
    "cfg3": dict(name="cfg3: LASP-2 masked layer fwd+bwd at Linear-Llama3-1B shape, B=1 H=16 d=128, N=524288 total",
                 n=524288, masked=True),
    # BASELINE.json configs[4]: the masked sequence-length sweep at 8 GPUs (64K ... 2M; --seq-len
    # picks the point, default the largest); N > 1 lines carry the comm / compute breakdown (`comm`)
    "cfg5": dict(name="cfg5: LASP-2 masked layer fwd+bwd, sequence-length sweep point, B=1 H=16 d=128, "
                      "N=2097152 total (64K-2M with --seq-len)",
                 n=2097152, masked=True),
    # LASP-2H N layer (K/V all_gather + causal softmax); opt-in (compute-bound, seconds per step at full N)
    "cfg4": dict(name="cfg4: LASP-2H causal softmax layer fwd+bwd (K/V AllGather), B=1 H=16 d=128, N=262144 total",
                 n=262144, masked=True, softmax=True),
}
BC = 256  # block size pinned for the algorithmic FLOP count


def flops_per_token(masked: bool, softmax: bool = False, n: int = 0) -> float:
    """Causal-useful algorithmic FLOPs per token (all heads), BASELINE.md §3.
    LASP-2H softmax: 7*d*N(N+1) per head for the whole layer -> 7*d*(N+1) per token."""
    if softmax:
        return float(7 * D * (n + 1) * H)
    per_head = 12 * D * D + (7 * D * (BC + 1) if masked else 0)
    return float(per_head * H)


def executed_flops_per_token(masked: bool, softmax: bool = False, n: int = 0) -> float:
    """FLOPs the kernels actually issue per token (all heads), SURVEY §8d's secondary column: 128-token
    blocks with full diagonal squares plus the recomputed products. Masked (default schedule):
    forward segment states 2d^2 + chunk pass 4d^2 + 4*128*d, backward dQ pass 6d^2 + 4*128*d and
    dK/dV pair 8d^2 + 8*128*d: 20d^2 + 2048d. Unmasked: 12d^2 (nothing recomputed). LASP-2H: the
    diagonal 128 x 128 blocks in full, 7d(N + 128)."""
    if softmax:
        return float(7 * D * (n + 128) * H)
    return float((20 * D * D + 16 * 128 * D if masked else 12 * D * D) * H)


def min_bytes_per_token() -> float:
    """fwd reads q,k,v writes o; bwd reads q,k,v,dO writes dq,dk,dv: 22*d bytes/token/head (bf16)."""
    return 22.0 * D * H


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return dict(hbm=j["hbm_gbs"], tensor=j["bf16_tflops"], tensor_sustained=j.get("bf16_tflops_sustained"),
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, tensor=1590.0, tensor_sustained=1400.0, source="fallback (B200_PROFILING.md)")


def ncu_traffic(workload: str, kernel_key: str):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture
    of this same bench command (profiles/ncu_traffic.json[workload][entry]), if present."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        rec = json.loads(p.read_text()).get(workload, {}).get(kernel_key)
        return None if rec is None else rec["bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """SM clock / throttle reasons sampled in-process through NVML every ~5 ms.

    Started before warm-up (so nothing spawns inside a timed region);
    summary(t0, t1) keeps only samples taken inside [t0, t1] (host clock).
    """

    # every NVML clocks-event reason bit (nvmlClocksEventReasons), so a clock below max is explained
    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
               "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

    def __init__(self, index: int, period: float = 0.005) -> None:
        self.index = index
        self.period = period
        self.samples: list[tuple[float, float, int, float]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        except Exception:  # noqa: BLE001 - reported as unsampled
            self._thread = None
        return self

    def _run(self):
        nv, h = self._nv, self._h
        try:
            self.power_limit_w = nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1e3
        except Exception:  # noqa: BLE001
            self.power_limit_w = None
        while not self._stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                try:
                    pw = nv.nvmlDeviceGetPowerUsage(h) / 1e3
                except Exception:  # noqa: BLE001
                    pw = float("nan")
                self.samples.append((time.time(), sm, rs, pw))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self, t0: float | None = None, t1: float | None = None) -> dict:
        rows = [r for r in self.samples if (t0 is None or r[0] >= t0) and (t1 is None or r[0] <= t1)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({n for *_, rs, _ in rows for n, bit in self.REASONS.items() if rs & bit} - {"gpu_idle"})
        bits = 0
        for r in rows:
            bits |= r[2]
        pw = [r[3] for r in rows if r[3] == r[3]]
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": min(r[1] for r in rows), "reasons": reasons, "samples": len(rows),
                "reason_bits_or": hex(bits),
                "reason_samples": {n: sum(1 for r in rows if r[2] & bit) for n, bit in self.REASONS.items()
                                   if any(r[2] & bit for r in rows)},
                "power_w_median": statistics.median(pw) if pw else None, "power_w_max": max(pw) if pw else None,
                "power_limit_w": getattr(self, "power_limit_w", None)}


# ---------------------------------------------------------------------------
# CPU reference arm / cpu_baseline: the oracle port on a bounded sample
# ---------------------------------------------------------------------------

def _oracle_inputs(workload: str, n: int, dtype):
    import numpy as np  # noqa: F401

    from oracle import lasp_oracle as O

    return tuple(O.gen_slots(0, B, H, n, D, t, dtype) for t in ("q", "k", "v", "do"))


def _oracle_iteration(workload: str, n: int, world: int, inputs):
    """One fwd+bwd iteration of the reference algorithm (the numpy oracle port restating
    lasp2.py:390-409 / standard_sp.py:112-127) on a world of `world` chunks."""
    from oracle import lasp_oracle as O

    wl = WORKLOADS[workload]
    q, k, v, do = inputs
    if wl.get("softmax"):
        return O.cp_full(q, k, v, do, world, True)
    return O.lasp2_full(q, k, v, do, world, wl["masked"], bc=BC)


# largest N the CPU port runs per workload (masked: the blocked intra pass is ~1.3 K tok/s per
# core-second; LASP-2H: the full softmax rows are O(N^2)); cfg2 runs at its full N
CPU_MAX_N = {"cfg2": 131072, "cfg3": 16384, "cfg4": 4096, "cfg5": 16384}


def _time_oracle(workload: str, n: int, world: int, dtype, iters: int, warmup: int = 1) -> dict:
    import numpy as np

    inputs = _oracle_inputs(workload, n, dtype)
    for _ in range(warmup):
        _oracle_iteration(workload, n, world, inputs)
    times = []
    for _ in range(max(1, iters)):
        t0 = time.perf_counter()
        _oracle_iteration(workload, n, world, inputs)
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return {"tokens_per_s": n / med, "ms_per_iteration": med * 1e3, "iterations": len(times),
            "dtype": np.dtype(dtype).name, "seq_len": n, "chunks": world}


def cpu_reference(workload: str, world: int = 1) -> dict:
    """cpu_baseline of the GPU line: the oracle port (f32, all host cores) on the same
    workload at its full N when the port can run it (cfg2), else at the largest N it runs
    in seconds (same B, H, d, T; labelled, not extrapolated). Adds the f64 number of the
    same sample and the cfg1 config exactly (B=1 H=4 d=64 N=4096 T=2 masked) in f32 / f64."""
    import numpy as np

    from oracle import lasp_oracle as O

    cores = len(os.sched_getaffinity(0))
    n = min(WORKLOADS[workload]["n"], CPU_MAX_N[workload])
    t0 = time.perf_counter()
    main = _time_oracle(workload, n, world, np.float32, iters=3)
    f64 = _time_oracle(workload, n, world, np.float64, iters=1, warmup=0)
    # cfg1 exactly (BASELINE.json configs[0]): the reference's own CPU-runnable case
    q, k, v, do = (O.gen_slots(0, 1, 4, 4096, 64, t) for t in ("q", "k", "v", "do"))
    cfg1 = {}
    for nm, dt in (("f32", np.float32), ("f64", np.float64)):
        xs = [x.astype(dt) for x in (q, k, v, do)]
        O.lasp2_full(*xs, 2, True, bc=BC)
        ts = []
        while len(ts) < 3:
            a = time.perf_counter()
            O.lasp2_full(*xs, 2, True, bc=BC)
            ts.append(time.perf_counter() - a)
        cfg1[nm] = {"tokens_per_s": 4096 / statistics.median(ts), "ms_per_iteration": statistics.median(ts) * 1e3}
    full = n == WORKLOADS[workload]["n"]
    return {"value": main["tokens_per_s"], "unit": UNIT, "cores": cores, "kind": "port",
            "same_config": full, "ms_per_iteration": main["ms_per_iteration"],
            "sample": (f"numpy oracle port (oracle/lasp_oracle.py restating "
                       f"{'standard_sp.py:37-76' if WORKLOADS[workload].get('softmax') else 'lasp2.py:208-285'}), "
                       f"f32, {'full' if full else 'reduced'} N={n} of the same B=1 H=16 d=128 layer, T={world}, "
                       f"median of {main['iterations']} timed fwd+bwd iterations (not extrapolated), "
                       f"OpenBLAS threads={os.environ.get('OPENBLAS_NUM_THREADS', 'all cores')}"),
            "f64": {"value": f64["tokens_per_s"], "ms_per_iteration": f64["ms_per_iteration"], "seq_len": n},
            "cfg1_exact": {"config": "B=1 H=4 d=64 N=4096 T=2 masked (BASELINE.json configs[0])", **cfg1},
            "wall_s": time.perf_counter() - t0}


def run_reference_arm(args) -> None:
    """--impl reference: the reference algorithm's CPU implementation (oracle port, all host
    threads) on this arm's exact config (cfg2: full N, T = --gpus chunks); rank 0 only."""
    import numpy as np

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    n_full = seq_override.get(args.workload, wl["n"])
    n = min(n_full, CPU_MAX_N[args.workload])
    world = args.gpus
    cores = len(os.sched_getaffinity(0))
    inputs = _oracle_inputs(args.workload, n, np.float32)
    for _ in range(args.warmup):
        _oracle_iteration(args.workload, n, world, inputs)
    t0 = time.perf_counter()
    times = []
    for _ in range(args.steps):
        a = time.perf_counter()
        _oracle_iteration(args.workload, n, world, inputs)
        times.append(time.perf_counter() - a)
    wall = time.perf_counter() - t0
    ms = statistics.mean(times) * 1e3
    v = n / (ms / 1e3)
    full = n == n_full
    sample = (f"numpy oracle port (oracle/lasp_oracle.py), f32, {'full' if full else 'reduced'} N={n}, "
              f"T={world} chunks, {args.steps} timed fwd+bwd iterations after {args.warmup} warm-up, "
              f"host threads={cores}")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference datagen SplitMix64 counter-hash)",
            "config": bench_config(args.workload, n, world, args.state_exchange, args.balanced),
            "same_config": full,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


def bench_config(workload: str, n: int, world: int, state_exchange: str, balanced: bool, fallback: str = "") -> dict:
    """The `config` object of both arms (identical keys and values for the same run)."""
    wl = WORKLOADS[workload]
    return {"workload": wl["name"], "global_batch": B, "seq_len": n, "chunk_per_gpu": n // world, "heads": H,
            "dim": D, "parallelism": f"sp{world}", "masked": wl["masked"],
            "l2": "inputs >= 2 GiB per step >> 126 MB L2; no flush needed",
            "state_exchange": (state_exchange if world > 1 else "none (one rank)") + (
                f" (fell back to collective: {fallback})" if fallback else ""),
            "lasp2h_schedule": "balanced" if balanced else "contiguous"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

seq_override: dict[str, int] = {}


# algorithmic HBM traffic per launch in units of one bf16 (B, H, C, d) tensor
ALGO_UNITS = {"lasp2_causal_chunk": 4, "lasp2_apply_state": 2, "lasp2_segment_states": 2, "lasp2_dkdv_chunk": 6,
              "lasp2_state_apply": 3, "lasp2_apply_state2": 4, "lasp2_backward_chunk": 7,
              "lasp2_dq_chunk": 5,  # dO, V, K, Q in, dQ out
              # world-of-one persistent kernels: K,V in + Q in, O out | Q,dO in, dQ out + V,K in, dK,dV out
              "lasp2_nomask_forward_local": 4, "lasp2_nomask_backward_local": 7,
              # T > 1: the same kernels split around the exchange (profiler labels per phase)
              "lasp2_nomask_forward_phase1": 2,   # K, V in -> M_t
              "lasp2_nomask_forward_phase2": 2,   # Q in, O out
              "lasp2_nomask_backward_phase1": 3,  # Q, dO in, dQ out (+ dM_t)
              "lasp2_nomask_backward_phase2": 4}  # V, K in, dK, dV out


def measure_workload(workload: str, ctx, rank: int, world: int, steps: int, warmup: int, device,
                     use_graph: bool = True) -> dict:
    import torch
    import torch.distributed as dist

    from paper_2502_07563_b200 import _lib
    from paper_2502_07563_b200.datagen import gen_slots_device
    from paper_2502_07563_b200.lasp2 import rank_backward, rank_forward

    from paper_2502_07563_b200.standard_sp import _cp_backward_rank, _cp_forward_rank

    wl = WORKLOADS[workload]
    n, masked, softmax = seq_override.get(workload, wl["n"]), wl["masked"], wl.get("softmax", False)
    c = n // world
    q, k, v, do = (gen_slots_device(0, B, H, c, D, t, torch.bfloat16, device=device, row_offset=rank * c)
                   for t in ("q", "k", "v", "do"))

    def layer(bq, bk, bv, bdo):
        if softmax:
            out, cache = _cp_forward_rank(ctx, bq, bk, bv, True)
            g = _cp_backward_rank(ctx, cache, bdo)
        else:
            out, cache = rank_forward(ctx, bq, bk, bv, masked=masked)
            g = rank_backward(ctx, cache, bdo)
        return out, g.dq, g.dk, g.dv

    def step():
        return layer(q, k, v, do)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.current_stream()
    with ClockSampler(device.index) as clocks:
        for _ in range(warmup):
            step()
        sync_all()

        # (1) per-kernel profile: launches queued behind a device sleep, so every
        #     CUDA-event bracket measures the kernel alone (no host gaps)
        prof_steps = max(1, min(steps, 10))
        _lib.PROFILER.reset(enabled=True)
        dev_events = getattr(ctx, "device_events", None)
        if dev_events is not None:
            dev_events.clear()
        torch.cuda._sleep(int(6e8))
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for _ in range(prof_steps):
            step()
        p1.record(stream)
        sync_all()
        durations = _lib.PROFILER.durations_ms()
        launches_per_step = _lib.PROFILER.launches / prof_steps
        _lib.PROFILER.reset(enabled=False)
        prof_step_ms = p0.elapsed_time(p1) / prof_steps
        # collectives on the side stream (DistRankContext marks issue / completion there):
        # device duration of each, and how much of the step the compute stream spent not
        # running this library's kernels (the exposed exchange + launch gaps)
        comm = None
        if world > 1 and dev_events is not None:
            issues = [ev for kind, ev in dev_events if kind == "all_gather_issue"]
            dones = [ev for kind, ev in dev_events if kind == "all_gather_complete"]
            ag = [a.elapsed_time(b) for a, b in zip(issues, dones)]
            comm = {"allgathers_per_step": len(ag) / prof_steps,
                    "allgather_device_ms_mean": statistics.mean(ag) if ag else None,
                    "allgather_device_ms_max": max(ag) if ag else None,
                    "profiled_step_ms": prof_step_ms,
                    "kernel_sum_ms": sum(sum(v2) for v2 in durations.values()) / prof_steps}
            comm["exposed_ms_per_step"] = max(0.0, prof_step_ms - comm["kernel_sum_ms"])
            dev_events.clear()

        # (2) capture one step as a CUDA graph (host launch overhead removed)
        graph = None
        if use_graph:
            try:
                s2 = torch.cuda.Stream()
                s2.wait_stream(stream)
                with torch.cuda.stream(s2):
                    step()
                stream.wait_stream(s2)
                sync_all()
                graph = torch.cuda.CUDAGraph()
                # thread-local capture: NCCL's watchdog thread may query events meanwhile
                with torch.cuda.graph(graph, capture_error_mode="thread_local" if world > 1 else "global"):
                    outs = step()
                for _ in range(3):
                    graph.replay()
                sync_all()
            except Exception as exc:  # noqa: BLE001 - fall back to eager, reported
                print(f"[bench] graph capture failed ({exc!r}); timing eager launches", file=sys.stderr)
                graph = None
        run = graph.replay if graph is not None else step

        # (3) timed region: K steps between barrier+synchronize brackets, max over ranks
        sync_all()
        h0 = time.time()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(steps):
            run()
        t1.record(stream)
        sync_all()
        h1 = time.time()
        ms = max_over_ranks(t0.elapsed_time(t1) / steps)
        clk = clocks.summary(h0, h1)

        # (4) end-to-end through the public API, pipelined over three streams with two
        #     buffer sets: H2D of step i+1 (pinned host -> HBM) || fwd+bwd of step i ||
        #     D2H of step i-1 (outputs and all three gradients -> pinned host).
        bufs = [(q, k, v, do), tuple(t.clone() for t in (q, k, v, do))]
        runners = []
        for bi, (bq, bk, bv, bdo) in enumerate(bufs):
            def make(bq=bq, bk=bk, bv=bv, bdo=bdo):
                return layer(bq, bk, bv, bdo)
            if graph is not None:
                if bi == 0:
                    runners.append((graph.replay, outs))
                else:
                    g2 = torch.cuda.CUDAGraph()
                    s3 = torch.cuda.Stream()
                    s3.wait_stream(stream)
                    with torch.cuda.stream(s3):
                        make()
                    stream.wait_stream(s3)
                    sync_all()
                    with torch.cuda.graph(g2, capture_error_mode="thread_local" if world > 1 else "global"):
                        outs2 = make()
                    runners.append((g2.replay, outs2))
            else:
                runners.append((make, None))
        host_in = [t.cpu().pin_memory() for t in (q, k, v, do)]
        host_out = [[torch.empty(q.shape, dtype=q.dtype, pin_memory=True) for _ in range(4)] for _ in range(2)]
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()  # noqa: E731
        h2d_done, comp_done, d2h_done = [ev(), ev()], [ev(), ev()], [ev(), ev()]
        # the pipeline fills once and drains once per measurement (one H2D and one D2H not
        # overlapped): 32 steps keep that to ~1/32 of the steady-state PCIe-bound period
        e2e_steps = max(4, min(2 * steps, 32))
        sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h2d_s)
        for i in range(e2e_steps):
            bi = i & 1
            if i >= 2:
                h2d_s.wait_event(comp_done[bi])  # inputs of set bi no longer read
            with torch.cuda.stream(h2d_s):
                for dst, src in zip(bufs[bi], host_in):
                    dst.copy_(src, non_blocking=True)
                h2d_done[bi].record(h2d_s)
            stream.wait_event(h2d_done[bi])
            if i >= 2:
                stream.wait_event(d2h_done[bi])  # outputs of set bi already copied out
            fn, static_outs = runners[bi]
            res = fn()
            res = static_outs if static_outs is not None else res
            comp_done[bi].record(stream)
            d2h_s.wait_event(comp_done[bi])
            with torch.cuda.stream(d2h_s):
                for dst, src in zip(host_out[bi], res):
                    dst.copy_(src, non_blocking=True)
                d2h_done[bi].record(d2h_s)
        stream.wait_stream(h2d_s)
        stream.wait_stream(d2h_s)
        e1.record(stream)
        sync_all()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)

    # dominant kernel (most device time per step) and its roofline
    per_kernel = {k2: sum(v2) / prof_steps for k2, v2 in durations.items()}
    # among the kernels with an algorithmic byte / FLOP count (a fold behind a gloo all_gather
    # can outlast every compute launch in the profiled pass, but it is not the path's kernel)
    rated = [k2 for k2 in per_kernel if k2 in ALGO_UNITS or k2.startswith("lasp2h_softmax")]
    dom = max(rated or per_kernel, key=per_kernel.get)
    dom_launch_ms = statistics.mean(durations[dom])
    unit_bytes = B * H * c * D * 2  # one bf16 (B,H,C,d) tensor
    algo_bytes = ALGO_UNITS.get(dom, 0) * unit_bytes
    # causal softmax useful FLOPs of one rank: queries [rC, (r+1)C) see keys <= position
    pairs = H * (c * rank * c + c * (c + 1) / 2)
    algo_flops = {"lasp2h_softmax_forward": 4 * D * pairs, "lasp2h_softmax_backward": 10 * D * pairs}.get(dom, 0)
    return dict(workload=workload, n=n, c=c, masked=masked, softmax=softmax, ms=ms, e2e_ms=e2e_ms, per_kernel_ms=per_kernel, dominant=dom,
                dom_launch_ms=dom_launch_ms, dom_algo_bytes=algo_bytes, dom_algo_flops=algo_flops, launches_per_step=launches_per_step,
                h2d=4 * q.numel() * q.element_size() * world, d2h=4 * q.numel() * q.element_size() * world,
                clocks=clk, e2e_steps=e2e_steps, graph=graph is not None,
                kernel_sum_ms=sum(per_kernel.values()), comm=comm)


def summarize(r: dict, world: int, peaks: dict) -> dict:
    tok_s = r["n"] / (r["ms"] / 1e3)
    flop_s = flops_per_token(r["masked"], r.get("softmax", False), r["n"]) * tok_s
    byte_s = min_bytes_per_token() * tok_s
    achieved = r["dom_algo_bytes"] / (r["dom_launch_ms"] / 1e3) / 1e9
    tensor_peak, peak_kind = peaks["tensor"], "burst"
    if r.get("softmax"):  # tensor-bound: useful FLOPs of the dominant kernel per launch
        achieved = r["dom_algo_flops"] / (r["dom_launch_ms"] / 1e3) / 1e12
        if r["dom_launch_ms"] >= 50.0 and peaks.get("tensor_sustained"):
            # a launch this long runs at the board's sustained (power-limited) clock
            tensor_peak, peak_kind = peaks["tensor_sustained"], "sustained"
    peak = tensor_peak if r.get("softmax") else peaks["hbm"]
    traffic_key = r["workload"] if world == 1 else f"{r['workload']}@C={r['c']}"
    return dict(
        value=tok_s, ms_per_step=r["ms"],
        tensor_tflops_per_gpu=flop_s / world / 1e12,
        tensor_frac_of_peak=flop_s / world / (peaks["tensor"] * 1e12),
        executed_tflops_per_gpu=executed_flops_per_token(r["masked"], r.get("softmax", False), r["n"]) * tok_s
        / world / 1e12,
        min_bytes_gbs_per_gpu=byte_s / world / 1e9,
        hbm_frac_of_peak=byte_s / world / (peaks["hbm"] * 1e9),
        per_kernel_ms_per_step=r["per_kernel_ms"],
        roofline={"kernel": r["dominant"], "bound": "tensor" if r.get("softmax") else "hbm", "achieved": achieved,
                  "peak": peak, "unit": "TFLOP/s" if r.get("softmax") else "GB/s",
                  "frac": achieved / peak, "traffic": ncu_traffic(traffic_key, r["dominant"]),
                  "peak_source": peaks["source"] + (f", {peak_kind} bf16 figure" if r.get("softmax") else ""),
                  "algorithmic_bytes_per_launch": r["dom_algo_bytes"], "avg_launch_ms": r["dom_launch_ms"]},
        e2e={"value": r["n"] / (r["e2e_ms"] / 1e3), "unit": UNIT, "h2d_bytes_per_step": r["h2d"],
             "d2h_bytes_per_step": r["d2h"], "ms_per_step": r["e2e_ms"], "steps": r["e2e_steps"],
             "path": ("pinned host inputs -> HBM, rank_forward + rank_backward (the per-rank public API) "
                      "replayed from a CUDA graph captured once (Python call overhead outside the timed "
                      "region), outputs and all three gradients -> pinned host; H2D / compute / D2H "
                      "pipelined over three streams with two buffer sets") if r["graph"] else
                     "pinned host inputs -> HBM, eager rank_forward + rank_backward, outputs + gradients -> host"},
        gpu_launches_per_step=r["launches_per_step"], clocks=r["clocks"], graph=r["graph"],
        kernel_sum_ms=r["kernel_sum_ms"], comm=r.get("comm"))


def run_gpu_arm(args) -> None:
    import torch

    if args.balanced:
        from paper_2502_07563_b200 import standard_sp as _sp
        _sp.BALANCED = True

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    local = local % torch.cuda.device_count()  # ranks may share a device (gloo smoke runs)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    from paper_2502_07563_b200 import comm

    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            # communicator-init lines (rank / nranks / transport) to stderr, so the JSON line
            # stays alone on stdout
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(args.dist_backend)
        peer = args.state_exchange == "peer"
        ctx = comm.DistRankContext(peer_exchange=peer,
                                   native_collectives=args.state_exchange == "native" and args.dist_backend == "nccl")
        if peer:  # fused state exchange over NVLink peer memory
            from paper_2502_07563_b200 import lasp2 as _l2
            _l2.STATE_EXCHANGE = "peer"
    else:
        ctx = comm.LocalRankContext()
    peaks = load_peaks()
    use_graph = not args.eager
    main = measure_workload(args.workload, ctx, rank, world, args.steps, args.warmup, device, use_graph)
    sec_name = "cfg3" if args.workload == "cfg2" else "cfg2"
    secondary = None if args.no_secondary else measure_workload(sec_name, ctx, rank, world, args.steps, args.warmup,
                                                                device, use_graph)
    if rank == 0:
        s = summarize(main, world, peaks)
        line = {"metric": METRIC, "value": s["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": s["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic: reference datagen (SplitMix64 counter-hash) generated on device, bf16",
                "config": bench_config(args.workload, main["n"], world, args.state_exchange, args.balanced,
                                       getattr(ctx, "peer_fallback", None) or ""),
                "tensor_frac_of_peak": s["tensor_frac_of_peak"], "tensor_tflops_per_gpu": s["tensor_tflops_per_gpu"],
                "executed_tflops_per_gpu": s["executed_tflops_per_gpu"],
                "hbm_frac_of_peak_min_bytes": s["hbm_frac_of_peak"], "roofline": s["roofline"],
                "e2e": s["e2e"], "gpu_launches": int(round(s["gpu_launches_per_step"] * args.steps)),
                "clocks": s["clocks"], "per_kernel_ms_per_step": s["per_kernel_ms_per_step"],
                "kernel_sum_ms_per_step": s["kernel_sum_ms"], "cuda_graph": s["graph"]}
        if s["comm"] is not None:
            line["comm"] = s["comm"]
        if secondary is not None:
            ss = summarize(secondary, world, peaks)
            line["secondary"] = {"workload": WORKLOADS[sec_name]["name"], "value": ss["value"], "unit": UNIT,
                                 "ms_per_step": ss["ms_per_step"], "chunk_per_gpu": secondary["c"],
                                 "tensor_frac_of_peak": ss["tensor_frac_of_peak"],
                                 "tensor_tflops_per_gpu": ss["tensor_tflops_per_gpu"],
                                 "executed_tflops_per_gpu": ss["executed_tflops_per_gpu"],
                                 "hbm_frac_of_peak_min_bytes": ss["hbm_frac_of_peak"], "roofline": ss["roofline"],
                                 "e2e": ss["e2e"], "per_kernel_ms_per_step": ss["per_kernel_ms_per_step"],
                                 "kernel_sum_ms_per_step": ss["kernel_sum_ms"], "clocks": ss["clocks"],
                                 "gpu_launches_per_step": ss["gpu_launches_per_step"], "comm": ss["comm"]}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_reference(args.workload, world)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--balanced", action="store_true",
                    help="cfg4 (LASP-2H): causal load balance across ranks (standard_sp.BALANCED)")
    ap.add_argument("--state-exchange", default="collective", choices=["collective", "peer", "native"],
                    help="N>1: torch.distributed NCCL all_gather of the states, the fused put into "
                         "symmetric-memory peers, or NCCL through the C ABI's wrappers (native)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of CUDA-graph replay")
    ap.add_argument("--seq-len", type=int, default=0, help="override N of the selected workload")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo for multi-rank smoke runs on one GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3 (timing rules)")
    if args.seq_len:
        seq_override[args.workload] = args.seq_len
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
