"""LASP-2H cfg4 at its 8-GPU per-rank shapes on one GPU, contiguous vs balanced
schedule (standard_sp.BALANCED): every rank's attention kernels (fwd + bwd) timed
in isolation, communication excluded. The layer time at 8 GPUs is bounded by the
slowest rank."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402
from paper_2502_07563_b200.standard_sp import _pairing  # noqa: E402

W, N, H, D = 8, 262144, 16, 128
C = N // W
per = H * C * D


def timeit(fn, iters=2):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


kf = torch.stack([gen_slots_device(0, 1, H, C, D, "k", row_offset=r * C).reshape(H * C, D) for r in range(W)])
vf = torch.stack([gen_slots_device(0, 1, H, C, D, "v", row_offset=r * C).reshape(H * C, D) for r in range(W)])
qs = [gen_slots_device(0, 1, H, C, D, "q", row_offset=t * C) for t in range(W)]
dos = [gen_slots_device(0, 1, H, C, D, "do", row_offset=t * C) for t in range(W)]
grads = torch.empty((W, 2, 1, H, C, D), dtype=torch.float32, device="cuda")


def unit(t, lo, hi, causal):
    """fwd + bwd of rank t's queries against keys [lo, hi) (key indices, rank-major layout)."""
    q, do = qs[t], dos[t]
    off = t * C - lo
    out, lse = ops.softmax_forward(q, kf, vf, causal, off if causal else 0, kv_tokens=hi - lo, kv_chunk=C,
                                   kv_rank_stride=per, kv_start=lo)

    def run():
        ops.softmax_forward(q, kf, vf, causal, off if causal else 0, kv_tokens=hi - lo, kv_chunk=C,
                            kv_rank_stride=per, kv_start=lo)
        ops.softmax_backward_acc(q, kf, vf, out, lse, do, causal, off if causal else 0, kv_tokens=hi - lo,
                                 kv_chunk=C, kv_rank_stride=per, grads=grads, grad_rank_stride=2 * per,
                                 dv_offset=per, key_range=True, kv_start=lo)
    return timeit(run)


plain = [unit(t, 0, (t + 1) * C, True) for t in range(W)]
bal = []
for t in range(W):
    helper, guest, u = _pairing(t, W, C, 128)  # u in keys (half chunks at even W)
    u = u if helper >= 0 else 0
    ms = unit(t, u, (t + 1) * C, True)
    if guest >= 0:
        ms += unit(guest, 0, _pairing(guest, W, C, 128)[2], False)
    bal.append(ms)
print("contiguous per-rank fwd+bwd ms:", [round(x, 1) for x in plain], f"-> max {max(plain):.1f}")
print("balanced   per-rank fwd+bwd ms:", [round(x, 1) for x in bal], f"-> max {max(bal):.1f}")
print(f"slowest-rank speed-up {max(plain) / max(bal):.2f}x")
