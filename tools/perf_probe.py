"""Quick per-kernel timing on one GPU (not the bench): bf16, H=16, d=128."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import lasp2, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402


def timeit(fn, iters=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
    h, d = 16, 128
    q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
    unit = h * n * d * 2 / 1e9  # GB per tensor
    nseg = ops.num_segments(k)
    print(f"N={n} H={h} d={d} nseg={nseg} tensor={unit:.3f} GB")
    seg = ops.segment_states(k, v, nseg)
    t = timeit(lambda: ops.segment_states(k, v, nseg))
    print(f"segment_states {t:.3f} ms  {2 * unit / t * 1e3:.0f} GB/s")
    t = timeit(lambda: ops.scan_segments(seg.clone(), False, k.dtype))
    print(f"scan(+clone) {t:.3f} ms")
    t = timeit(lambda: ops.causal_chunk(q, k, v, seg, None, nseg))
    print(f"causal_chunk {t:.3f} ms  {4 * unit / t * 1e3:.0f} GB/s")
    t = timeit(lambda: ops.dkdv_chunk(q, k, v, do, seg, None, nseg))
    print(f"dkdv_chunk (pair) {t:.3f} ms  {6 * unit / t * 1e3:.0f} GB/s")
    m = torch.randn((1, h, d, d), device="cuda")
    t = timeit(lambda: ops.apply_state(q, m))
    print(f"apply_state {t:.3f} ms  {2 * unit / t * 1e3:.0f} GB/s")

    class Ctx:
        sp_position, sp_size = 0, 1

        def all_gather(self, p, tag=""):
            return p.unsqueeze(0)

        def all_gather_async(self, p, tag=""):
            class P:
                def wait(s):
                    return p.unsqueeze(0)
            return P()

        def mark(self, *a):
            pass

    ctx = Ctx()

    def step():
        out, cache = lasp2._forward_masked_rank(ctx, q, k, v)
        lasp2._backward_masked_rank(ctx, cache, do)

    t = timeit(step, 3)
    flops = (12 * d * d + 7 * d * 257) * h * n
    print(f"masked fwd+bwd {t:.3f} ms  {n / t * 1e3:.0f} tok/s  {flops / t / 1e9:.1f} TFLOP/s "
          f"{22 * d * h * n / t / 1e6:.0f} GB/s(min-bytes)")

    def step_u():
        out, cache = lasp2._forward_nomask_rank(ctx, q, k, v)
        lasp2._backward_nomask_rank(ctx, cache, do)

    t = timeit(step_u, 3)
    print(f"unmasked fwd+bwd {t:.3f} ms  {n / t * 1e3:.0f} tok/s {22 * d * h * n / t / 1e6:.0f} GB/s(min-bytes)")


if __name__ == "__main__" and not (len(sys.argv) > 2 and sys.argv[2] == "softmax"):
    main()


def softmax_probe(n=32768, h=16, d=128):
    """Causal softmax attention (one rank, W=1) fwd and bwd throughput."""
    q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
    per = h * n * d
    out, lse = ops.softmax_forward(q, k, v, True, 0, n, n, 0)
    t = timeit(lambda: ops.softmax_forward(q, k, v, True, 0, n, n, 0), 3)
    fl_fwd = 4 * d * n * (n + 1) / 2 * h  # causal-useful: 2 GEMMs x 2 flop
    print(f"softmax fwd N={n} H={h}: {t:.3f} ms  {fl_fwd / t / 1e9:.1f} TFLOP/s")
    grads = torch.empty((1, 2, 1, h, n, d), dtype=torch.float32, device="cuda")
    t = timeit(lambda: ops.softmax_backward(q, k, v, out, lse, do, True, 0, n, n, 0, grads, 0, per), 3)
    fl_bwd = 10 * d * n * (n + 1) / 2 * h  # 5 GEMMs (S recompute, dP, dV, dK, dQ)
    print(f"softmax bwd N={n} H={h}: {t:.3f} ms  {fl_bwd / t / 1e9:.1f} TFLOP/s (5-GEMM count)")


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "softmax":
    softmax_probe(int(sys.argv[3]) if len(sys.argv) > 3 else 32768)
