"""Fused peer state exchange across PROCESSES on one GPU: 2 ranks over gloo, torch
symmetric memory (CUDA IPC mappings of the same device), lasp2.STATE_EXCHANGE = "peer":
masked and unmasked fwd+bwd against the oracle. Prints whether the rendezvous held."""
import os
import socket
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import lasp_oracle as O  # noqa: E402


def worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_07563_b200 import lasp2
        from paper_2502_07563_b200.comm import DistRankContext

        lasp2.STATE_EXCHANGE = "peer"
        res = {}
        for masked in (True, False):
            n, d, h = 512 * world, 64, 2
            x = O.inputs(n, d, 1, h, 7)
            x = [O.bf16_round(a) for a in x]
            c = n // world
            qc, kc, vc, dc = (torch.from_numpy(np.ascontiguousarray(a[:, :, rank * c:(rank + 1) * c])).to(
                "cuda", torch.bfloat16) for a in x)
            ctx = DistRankContext(peer_exchange=True)
            o, cache = lasp2.rank_forward(ctx, qc, kc, vc, masked=masked)
            g = lasp2.rank_backward(ctx, cache, dc)
            torch.cuda.synchronize()
            res[masked] = ([t.double().cpu().numpy() for t in (o, g.dq, g.dk, g.dv)], ctx.peer_fallback or ctx.peer_method,
                           ctx.stats.allgather_launches)
        q.put((rank, res))
    except Exception as exc:  # noqa: BLE001
        import traceback

        q.put((rank, f"{exc!r}\n{traceback.format_exc()}"))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        if isinstance(out[r], str):
            print(f"rank {r} failed: {out[r]}")
            sys.exit(1)
    n, d, h = 512 * world, 64, 2
    x = [O.bf16_round(a) for a in O.inputs(n, d, 1, h, 7)]
    for masked in (True, False):
        ref = O.lasp2_full(*x, world, masked)
        got = [np.concatenate([out[r][masked][0][i] for r in range(world)], axis=2) for i in range(4)]
        errs = [O.normalized_error(g, rr) for g, rr in zip(got, ref)]
        print(f"masked={masked}: peer method / fallback {[out[r][masked][1] for r in range(world)]}, "
              f"all_gather ledger {[out[r][masked][2] for r in range(world)]}, normalised errors "
              + " ".join(f"{e:.2e}" for e in errs))
