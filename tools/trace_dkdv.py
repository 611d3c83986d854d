"""Timeline of one CTA (rank 0, dK) of the dK/dV pair kernel (clock64 trace points)."""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_2502_07563_b200 import _lib, ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402

NAMES = {10: "mma:wait_qk", 11: "mma:qk_landed", 12: "mma:p_prev_ok", 13: "mma:sst_ok", 14: "mma:o_empty_ok",
         15: "mma:v_landed", 16: "mma:p_ok", 20: "epi:wait_s", 21: "epi:s_full", 22: "epi:stg_free", 23: "epi:p_done",
         24: "epi:st_full", 25: "epi:sst_done", 26: "epi:o_full", 27: "epi:o_stored"}

n = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
h, d = 16, 128
q, k, v, do = (gen_slots_device(0, 1, h, n, d, t) for t in ("q", "k", "v", "do"))
nseg = ops.num_segments(k)
seg = ops.segment_states(k, v, nseg)
buf = torch.zeros(128, dtype=torch.int64, device="cuda")
ops.dkdv_chunk(q, k, v, do, seg, None, nseg)
torch.cuda.synchronize()
_lib.call("lasp2_debug_trace", buf.data_ptr())
ops.dkdv_chunk(q, k, v, do, seg, None, nseg)
torch.cuda.synchronize()
_lib.call("lasp2_debug_trace", None)
raw = [x & ((1 << 64) - 1) for x in buf.cpu().tolist() if x != 0]
rec = [((x >> 56) & 0xFF, (x >> 48) & 0xFF, x & 0xFFFFFFFFFFFF) for x in raw]
t0 = min(r[2] for r in rec)
by_blk = defaultdict(dict)
for ev, blk, clk in rec:
    by_blk[blk].setdefault(ev, clk - t0)
blocks = sorted(by_blk)
print("block period (epi:p_done deltas):", [by_blk[b + 1].get(23, 0) - by_blk[b].get(23, 0) for b in blocks[:-1]])
for b in blocks[2:6]:
    print(f"--- block {b}")
    for ev, c in sorted(by_blk[b].items(), key=lambda x: x[1]):
        print(f"   {c:10d}  {NAMES.get(ev, ev)}")
