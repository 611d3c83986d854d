"""LASP-2H cfg4 at its 8-GPU per-rank shape on one GPU: the slowest rank (t = 7)
of N = 262144, W = 8 (C = 32768 queries at row offset 7C against all 262144
gathered keys, rank-major as the all_gather leaves them), H = 16, d = 128, bf16.
Forward + backward kernel time and causal-useful TFLOP/s (4d / 10d FLOP per
visible query-key pair)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

W, N, H, D = 8, 262144, 16, 128
T = int(sys.argv[1]) if len(sys.argv) > 1 else W - 1
C = N // W


def timeit(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


q, do = (gen_slots_device(0, 1, H, C, D, tag, row_offset=T * C) for tag in ("q", "do"))
# gathered K / V, rank-major [W][B*H*C][d]: rank r's chunk = rows [rC, (r+1)C) of every slot
kf = torch.stack([gen_slots_device(0, 1, H, C, D, "k", row_offset=r * C).reshape(H * C, D) for r in range(W)])
vf = torch.stack([gen_slots_device(0, 1, H, C, D, "v", row_offset=r * C).reshape(H * C, D) for r in range(W)])
stride = H * C * D
out, lse = ops.softmax_forward(q, kf, vf, True, T * C, kv_tokens=N, kv_chunk=C, kv_rank_stride=stride)
pairs = H * (C * T * C + C * (C + 1) / 2)
tf = timeit(lambda: ops.softmax_forward(q, kf, vf, True, T * C, kv_tokens=N, kv_chunk=C, kv_rank_stride=stride))
grads = torch.empty((W, 2, 1, H, C, D), dtype=torch.float32, device="cuda")
tb = timeit(lambda: ops.softmax_backward(q, kf, vf, out, lse, do, True, T * C, N, C, stride, grads, 2 * stride,
                                         stride))
print(f"cfg4 rank {T}/{W}: C={C} keys={(T + 1) * C}  fwd {tf:.2f} ms {4 * D * pairs / tf / 1e9:.0f} TFLOP/s  "
      f"bwd {tb:.2f} ms {10 * D * pairs / tb / 1e9:.0f} TFLOP/s  layer {tf + tb:.2f} ms")
