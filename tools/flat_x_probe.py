"""cfg2's unmasked layer per rank at chunk C in a T-rank world: the all_gather path (phase 1,
[exchange], fold, phase 2 per direction: 6 launches) against the fused-exchange kernels
(lasp2_nomask_forward_x / backward_x: 2 launches). The other T-1 ranks are complete in advance
(their receive slots and flags filled, tests/test_gpu_flat_exchange.py), so this times one
rank's device work; the all_gather itself is a local copy on the unfused side. CUDA graphs.

usage: python tools/flat_x_probe.py [C] [T]"""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2502_07563_b200 import ops  # noqa: E402
from paper_2502_07563_b200.datagen import gen_slots_device  # noqa: E402
from test_gpu_flat_exchange import _world  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rank = world - 1
q, k, v, do = (gen_slots_device(0, 1, 16, c, 128, t, row_offset=rank * c) for t in ("q", "k", "v", "do"))
like = torch.empty((1, 16, 128, 128), dtype=torch.float32, device="cuda")
others = torch.randn((world, 1, 16, 128, 128), device="cuda")
fx, *keep_f = _world(rank, world, like, others)  # keep the fake peers' buffers alive (the tables point there)
bx, *keep_b = _world(rank, world, like, others)


def unfused():
    m_t = ops.nomask_forward_phase(q, k, v, torch.empty_like(like), 1)
    g = others.clone()
    g[rank] = m_t
    m = ops.sum_states(g)
    out = ops.nomask_forward_phase(q, k, v, m, 2)
    dq, dm_t = ops.nomask_backward_phase1(q, do, m)
    g2 = others.clone()
    g2[rank] = dm_t
    dk, dv = ops.nomask_backward_phase2(v, k, ops.sum_states(g2))
    return out, dq, dk, dv


def fused():
    out, m = ops.nomask_forward_x(q, k, v, fx)
    dq, dk, dv = ops.nomask_backward_x(q, k, v, do, m, bx)
    return out, dq, dk, dv


def graph_ms(fn, reps=50):
    for _ in range(3):
        fn()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        gr.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


unit = 16 * c * 128 * 2 / 1e9
for name, fn in (("all_gather path", unfused), ("fused exchange", fused), ("all_gather path", unfused),
                 ("fused exchange", fused)):
    ms = graph_ms(fn)
    print(f"C={c} T={world} rank={rank} {name:16s} graph step {ms * 1e3:7.1f} us = {11 * unit / ms * 1e3:5.0f} GB/s "
          f"minimal bytes, {c / ms * 1e3 / 1e6:5.1f} M tok/s/GPU")


# per-CTA globaltimer timeline of one fused forward launch (lasp2_debug_trace)
from paper_2502_07563_b200 import _lib  # noqa: E402
buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
names = {0: "start", 1: "p1_done", 2: "barrier1", 3: "reduced+put", 7: "barrier2", 4: "flags+fold+barrier3",
         5: "p2_done", 6: "end"}
for label, fn in (("fwd_x", lambda: ops.nomask_forward_x(q, k, v, fx)),
                  ("bwd_x", lambda: ops.nomask_backward_x(q, k, v, do, like.new_zeros(like.shape), bx))):
    buf.zero_()
    torch.cuda.synchronize()
    _lib.call("lasp2_debug_trace", buf.data_ptr())
    fn()
    torch.cuda.synchronize()
    _lib.call("lasp2_debug_trace", None)
    t = buf.view(148, 8).cpu()
    t0 = t[:, 0][t[:, 0] > 0].min().item()
    print(f"--- {label} (us from the first CTA start): min / median / max over CTAs")
    for i in (0, 1, 2, 3, 7, 4, 5, 6):
        col = t[:, i]
        col = col[col > 0].double() - t0
        if col.numel():
            print(f"   {names[i]:20s} {col.min().item()/1e3:8.1f} {col.median().item()/1e3:8.1f} {col.max().item()/1e3:8.1f}")
