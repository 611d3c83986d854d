"""Timeline of one CTA (key block 0 of slot 0... the first CTA) of the LASP-2H backward (LASP2_TRACE build)."""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

NAMES = {10: "mma:blk_start", 11: "mma:ds_ready", 12: "mma:dvdkdq_issued", 13: "mma:dp_next_issued",
         14: "mma:s_next_issued", 20: "sm:wait_sdp", 21: "sm:sdp_full", 22: "sm:ds_done", 23: "sm:dq_full",
         24: "sm:dq_reduced"}
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
print("period (sm:ds_done deltas):", [by_blk[b + 1].get(22, 0) - by_blk[b].get(22, 0) for b in blocks[:-1]])
for b in blocks[2:5]:
    print(f"--- query block {b}")
    for ev, c in sorted(by_blk[b].items(), key=lambda x: x[1]):
        print(f"   {c:10d}  {NAMES.get(ev, ev)}")
