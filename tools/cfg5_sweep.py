"""cfg5 on one GPU: the LASP-2 masked layer's per-rank program at the 8-GPU
chunk sizes of the sequence-length sweep (N = 64K ... 2048K, W = 8, C = N/8,
B=1 H=16 d=128 bf16), for the first (t = 0) and last (t = 7) rank, in the
sequential and the overlap schedule, with the state all_gather replaced by a
local copy into a [W, ...] buffer (the other ranks' states are fixed
synthetic values). Reports per-rank device time of forward and backward, the
compute before / after each exchange (what an all_gather of 1 MiB would be
exposed against or hidden behind), and the per-GPU throughput this implies
with the exchange itself costed at 0 (it is not measurable on one GPU; NCCL
all_gather of 1 MiB over NVLink is O(10-20 us)).

    python tools/cfg5_sweep.py [N ...]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import comm, lasp2  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

import os  # noqa: E402

W, H, D = 8, 16, 128
if os.environ.get("GATHERED_FUSED"):  # A/B: consumers fold the gathered states in their prologue
    lasp2.GATHERED_FUSED_CONSUMER = True
if os.environ.get("NSEG"):  # A/B: segments per slot of the masked passes
    from paper_2502_07563_b200 import ops  # noqa: E402
    ops.num_segments = lambda x, _n=int(os.environ["NSEG"]): _n
MASKED = "--unmasked" not in sys.argv  # --unmasked: cfg2's layer at its W = 8 chunk (N = 128K -> C = 16K)
SIZES = [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [65536, 131072, 262144, 524288, 1048576, 2097152]


class ProbeCtx(comm.LocalRankContext):
    """Rank t of a W-rank SP group; all_gather = copy into slot t of a fixed buffer."""

    def __init__(self, t: int, world: int) -> None:
        super().__init__()
        self.sp_position, self.sp_size, self.rank = t, world, t
        self.bufs: dict[tuple, torch.Tensor] = {}
        self.events: list[tuple[str, torch.cuda.Event]] = []

    def all_gather_async(self, payload, tag=""):
        key = (tag, tuple(payload.shape), payload.dtype)
        buf = self.bufs.get(key)
        if buf is None:
            g = torch.Generator(device=payload.device).manual_seed(len(self.bufs))
            buf = (torch.rand((self.sp_size, *payload.shape), generator=g, device=payload.device) - 0.5)
            buf = (buf * payload.abs().max().clamp_min(1e-3)).to(payload.dtype)
            self.bufs[key] = buf
        self.mark(f"ag_issue:{tag}")
        buf[self.sp_position].copy_(payload)
        self.mark(f"ag_done:{tag}")

        class _Done:
            def wait(self_inner):
                return buf

        return _Done()

    def mark(self, kind, detail=""):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append((kind, ev))


def run(n: int, t: int, overlap: bool, iters: int = 5):
    c = n // W
    q, k, v, do = (gen_slots_device(0, 1, H, c, D, tag, row_offset=t * c) for tag in ("q", "k", "v", "do"))
    ctx = ProbeCtx(t, W)

    def step():
        ctx.events.clear()
        ctx.mark("start")
        if MASKED:
            out, cache = lasp2._forward_masked_rank(ctx, q, k, v, overlap=overlap)
        else:
            out, cache = lasp2._forward_nomask_rank(ctx, q, k, v)
        ctx.mark("fwd_end")
        (lasp2._backward_masked_rank if MASKED else lasp2._backward_nomask_rank)(ctx, cache, do)
        ctx.mark("bwd_end")
        return out

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    acc: dict[str, float] = {}
    for _ in range(iters):
        step()
        torch.cuda.synchronize()
        t0 = ctx.events[0][1]
        seen: dict[str, int] = {}
        for kind, ev in ctx.events[1:]:
            i = seen.get(kind, 0)
            seen[kind] = i + 1
            key = f"{kind}#{i}"
            acc[key] = acc.get(key, 0.0) + t0.elapsed_time(ev) / iters
    # the same step captured in a CUDA graph (how bench.py runs it): no launch gaps
    ctx.mark = lambda kind, detail="": None
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    graph.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters * 4):
        graph.replay()
    b.record()
    torch.cuda.synchronize()
    acc["graph_step"] = a.elapsed_time(b) / (iters * 4)
    return c, acc


def main() -> None:
    print(f"per-rank sweep, W={W} H={H} d={D} bf16 {'masked' if MASKED else 'unmasked'}; "
          "exchange = local copy (0 cost)")
    for n in SIZES:
        for overlap in ((False, True) if MASKED else (False,)):
            for t in (0, W - 1):
                c, ev = run(n, t, overlap)
                fwd, step = ev["fwd_end#0"], ev["bwd_end#0"]
                ag1 = ev["ag_issue:state#0"]
                ag2 = ev.get("ag_issue:state_grad#0", float("nan"))
                intra = ev.get("intra_end#0", float("nan")) - ev.get("intra_start#0", float("nan"))
                ag2 = ag2 if MASKED else ev.get("ag_issue:state_grad#0", float("nan"))
                flops = (12 * D * D + (7 * D * 257 if MASKED else 0)) * H * c  # BASELINE.md §3, per rank
                print(f"N={n:>8} C={c:>7} {'overlap   ' if overlap else 'sequential'} t={t}: "
                      f"fwd {fwd:7.3f} ms (compute before AG {ag1:6.3f}, intra {intra:6.3f}) "
                      f"bwd {step - fwd:7.3f} ms (before dM AG {ag2 - fwd:6.3f}) step {step:7.3f} ms  "
                      f"{c / step / 1e3:8.2f} M tok/s/GPU  {n / step / 1e3:8.1f} M tok/s x{W}  "
                      f"{flops / step / 1e9:6.0f} TFLOP/s/GPU")
                g = ev["graph_step"]
                print(f"{'':>27}graph-captured step {g:7.3f} ms  {c / g / 1e3:8.2f} M tok/s/GPU  "
                      f"{n / g / 1e3:8.1f} M tok/s x{W}  {flops / g / 1e9:6.0f} TFLOP/s/GPU  "
                      f"{22 * D * H * c / g / 1e6:6.0f} GB/s minimal-bytes")


if __name__ == "__main__":
    main()
