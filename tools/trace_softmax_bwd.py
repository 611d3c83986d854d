"""Timeline of CTA (0, 0) of the LASP-2H backward (tc_softmax_bwd3_kernel, LASP2_TRACE build):
MMA-warp and softmax-warp events per query block, clock64 cycles."""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

NAMES = {10: "mma:iter_start", 11: "mma:S_next_issued(r0_free)", 12: "mma:dP_next_issued(r1_free)",
         13: "mma:pds_ready", 14: "mma:dKdVdQ_issued", 20: "sm:s_full", 21: "sm:P_done", 22: "sm:dp_full",
         23: "sm:pds_arrive", 25: "sm:r1_free(prev dQ read)", 26: "sm:prev_dq_reduce_issued",
         27: "sm:dS_done", 28: "sm:image_free"}
n, h, d = 32768, 16, 128
q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
out, lse = ops.softmax_forward(q, k, v, True, 0, n, n, 0)
grads = torch.empty((1, 2, 1, h, n, d), dtype=torch.float32, device="cuda")
per = h * n * d
buf = torch.zeros(128, dtype=torch.int64, device="cuda")
ops.softmax_backward(q, k, v, out, lse, do, True, 0, n, n, 0, grads, 0, per)
torch.cuda.synchronize()
_lib.call("lasp2_debug_trace", buf.data_ptr())
ops.softmax_backward(q, k, v, out, lse, do, True, 0, n, n, 0, grads, 0, per)
torch.cuda.synchronize()
_lib.call("lasp2_debug_trace", None)
raw = [x & ((1 << 64) - 1) for x in buf.cpu().tolist() if x != 0]
rec = [((x >> 56) & 0xFF, (x >> 48) & 0xFF, x & 0xFFFFFFFFFFFF) for x in raw]
t0 = min(r[2] for r in rec)
by_blk = defaultdict(dict)
for ev, blk, clk in rec:
    by_blk[blk].setdefault(ev, clk - t0)
blocks = sorted(by_blk)
print("period (sm:pds_arrive deltas):", [by_blk[b + 1].get(23, 0) - by_blk[b].get(23, 0) for b in blocks[:-1]])
for b in blocks[2:6]:
    print(f"--- query block {b}")
    for ev, c in sorted(by_blk[b].items(), key=lambda x: x[1]):
        print(f"   {c:10d}  {NAMES.get(ev, ev)}")
