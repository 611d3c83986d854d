"""Timeline of the last query-tile CTA of the LASP-2H forward (LASP2_TRACE build)."""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

NAMES = {50: "mma:PV_A issued", 51: "mma:S_A issued", 52: "mma:PV_B issued", 53: "mma:S_B issued",
         60: "smA:s_full", 61: "smA:p_ready", 62: "smB:s_full", 63: "smB:p_ready"}
n, h, d = 32768, 16, 128
q, k, v = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v"))
buf = torch.zeros(256, dtype=torch.int64, device="cuda")
ops.softmax_forward(q, k, v, True, 0, n, n, 0)
torch.cuda.synchronize()
_lib.call("lasp2_debug_trace", buf.data_ptr())
ops.softmax_forward(q, k, v, True, 0, n, n, 0)
torch.cuda.synchronize()
_lib.call("lasp2_debug_trace", None)
raw = [x & ((1 << 64) - 1) for x in buf.cpu().tolist() if x != 0]
rec = [((x >> 56) & 0xFF, (x >> 48) & 0xFF, x & 0xFFFFFFFFFFFF) for x in raw]
t0 = min(r[2] for r in rec)
by_blk = defaultdict(dict)
for ev, blk, clk in rec:
    by_blk[blk].setdefault(ev, clk - t0)
blocks = sorted(by_blk)
print("period (smA:p_ready deltas):", [by_blk[b + 1].get(61, 0) - by_blk[b].get(61, 0) for b in blocks[:-1]])
allev = sorted(((c, b, ev) for b in blocks for ev, c in by_blk[b].items()))
for c, b, ev in allev:
    if 18 <= b <= 21:
        print(f"   {c:10d}  j={b:3d}  {NAMES.get(ev, ev)}")
