"""The product's per-rank programs in separate processes (reference comm.py:465-531
world semantics, one process per rank as under torchrun), all on cuda:0.

2 and 4 processes join a gloo group (NCCL refuses several ranks on one GPU; the
DistRankContext stages device payloads through the host for gloo) and run
exactly what bench.py and a model run per rank:

* ``lasp2.rank_forward`` / ``rank_backward`` (masked and unmasked, reference
  lasp2.py:208-285) — the tcgen05 kernels in bf16 and the validation kernels in
  f64, the state all_gathers and folds through DistRankContext;
* ``standard_sp._cp_forward_rank`` / ``_cp_backward_rank`` (LASP-2H, reference
  standard_sp.py:37-76) with contiguous chunks and with the balanced schedule
  (P2P send / recv between paired ranks), one reduce_scatter of dK / dV;
* ``lasp1.rank_forward`` / ``rank_backward`` (the ring, P2P);
* the fused peer state exchange (``lasp2.STATE_EXCHANGE = "peer"``)
  across processes: receive buffers, flags and acks mapped into every rank with
  CUDA IPC (torch symmetric memory refuses ranks sharing one device), the scan
  kernel's stores and the bf16 consumers' in-kernel flag waits crossing process
  boundaries — bitwise equal to the all_gather path.

The gathered results are compared with the oracle (reference tolerances in f64;
normalised <= 1e-2 for bf16 on the same bf16-rounded inputs, SURVEY §8a note P)
and the per-rank ledgers with the reference's launch counts.
"""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import lasp_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _chunk(x: np.ndarray, world: int, rank: int, dtype) -> torch.Tensor:
    c = x.shape[2] // world
    return torch.from_numpy(np.ascontiguousarray(x[:, :, rank * c:(rank + 1) * c])).to("cuda", dtype)


def _np(t: torch.Tensor) -> np.ndarray:
    return t.double().cpu().numpy()


CASES = {
    # name: (n, d, b, h, seed) -- f64 small enough for the oracle's reference tolerances,
    # bf16 at 256+ tokens per rank so every rank runs the tcgen05 path with several blocks
    "f64": (64, 16, 1, 2, 21),
    "bf16": (1024, 64, 1, 2, 22),
}


def _worker(rank, world, port, results):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_07563_b200 import lasp1, lasp2, standard_sp
        from paper_2502_07563_b200.comm import DistRankContext

        out = {}
        for name, (n, d, b, h, seed) in CASES.items():
            dt = torch.float64 if name == "f64" else torch.bfloat16
            q, k, v, do = O.inputs(n * world, d, b, h, seed)
            if name == "bf16":
                q, k, v, do = (O.bf16_round(x) for x in (q, k, v, do))
            qc, kc, vc, dc = (_chunk(x, world, rank, dt) for x in (q, k, v, do))
            for masked in (True, False):
                ctx = DistRankContext()
                o, cache = lasp2.rank_forward(ctx, qc, kc, vc, masked=masked)
                g = lasp2.rank_backward(ctx, cache, dc)
                torch.cuda.synchronize()
                out[f"lasp2_{name}_{masked}"] = [_np(x) for x in (o, g.dq, g.dk, g.dv)]
                out[f"lasp2_{name}_{masked}_ledger"] = (ctx.stats.allgather_launches, ctx.stats.p2p_sends)
                # the fused state exchange: the scan kernel stores M_t into every
                # rank's receive buffer through CUDA IPC mappings (symmetric memory refuses ranks
                # sharing a device) and the bf16 consumers wait for the flags inside their kernels
                lasp2.STATE_EXCHANGE = "peer"
                try:
                    ctx = DistRankContext(peer_exchange=True)
                    o, cache = lasp2.rank_forward(ctx, qc, kc, vc, masked=masked)
                    g = lasp2.rank_backward(ctx, cache, dc)
                    torch.cuda.synchronize()
                finally:
                    lasp2.STATE_EXCHANGE = "collective"
                out[f"peer_{name}_{masked}"] = [_np(x) for x in (o, g.dq, g.dk, g.dv)]
                out[f"peer_{name}_{masked}_info"] = (ctx.peer_method, ctx.peer_fallback, ctx.stats.allgather_launches)
                # the same program captured once in a CUDA graph and replayed: the epoch lives on
                # the device, so every replay is a new exchange (flags, acks, receive halves)
                lasp2.STATE_EXCHANGE = "peer"
                try:
                    side = torch.cuda.Stream()
                    side.wait_stream(torch.cuda.current_stream())
                    graph = torch.cuda.CUDAGraph()
                    with torch.cuda.stream(side):
                        with torch.cuda.graph(graph, stream=side):
                            o, cache = lasp2.rank_forward(ctx, qc, kc, vc, masked=masked)
                            g = lasp2.rank_backward(ctx, cache, dc)
                    torch.cuda.current_stream().wait_stream(side)
                    replays = []
                    for _ in range(3):
                        graph.replay()
                        torch.cuda.synchronize()
                        replays.append([_np(x) for x in (o, g.dq, g.dk, g.dv)])
                finally:
                    lasp2.STATE_EXCHANGE = "collective"
                out[f"peer_graph_{name}_{masked}"] = replays
                out[f"peer_graph_{name}_{masked}_epoch"] = [int(e.ep.item()) for e in ctx._exchanges.values()]
            for balanced in (False, True):
                standard_sp.BALANCED = balanced
                ctx = DistRankContext()
                o, cache = standard_sp._cp_forward_rank(ctx, qc, kc, vc, True)
                g = standard_sp._cp_backward_rank(ctx, cache, dc)
                torch.cuda.synchronize()
                out[f"cp_{name}_{balanced}"] = [_np(x) for x in (o, g.dq, g.dk, g.dv)]
                out[f"cp_{name}_{balanced}_ledger"] = (ctx.stats.allgather_launches,
                                                       ctx.stats.reduce_scatter_launches, ctx.stats.p2p_sends)
            standard_sp.BALANCED = False
            ctx = DistRankContext()
            o, cache = lasp1.rank_forward(ctx, qc, kc, vc, masked=True)
            g = lasp1.rank_backward(ctx, cache, dc)
            torch.cuda.synchronize()
            out[f"lasp1_{name}"] = [_np(x) for x in (o, g.dq, g.dk, g.dv)]
            out[f"lasp1_{name}_ledger"] = (ctx.stats.p2p_sends, ctx.stats.allgather_launches)
        results[rank] = out
    except Exception as exc:  # noqa: BLE001 - surfaced by the parent
        import traceback

        results[rank] = {"error": f"{exc!r}\n{traceback.format_exc()}"}
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module", params=[2, 4])
def world_results(request):
    import torch.multiprocessing as mp

    world = request.param
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    res = dict(results)
    for r in range(world):
        assert "error" not in res[r], res[r].get("error")
    return world, res


def _cat(res, world, key):
    return [np.concatenate([res[r][key][i] for r in range(world)], axis=2) for i in range(4)]


def _check(name, got, ref):
    names = ("out", "dq", "dk", "dv")
    if name == "f64":
        assert np.max(np.abs(got[0] - ref[0])) <= 1e-10  # lasp2.py forward tolerance
        for nm, g, r in zip(names[1:], got[1:], ref[1:]):
            assert O.relative_error(g, r) <= 1e-10, nm
    else:
        for nm, g, r in zip(names, got, ref):
            assert O.normalized_error(g, r) <= 1e-2, nm


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("masked", [True, False])
def test_lasp2_rank_programs_match_oracle(world_results, name, masked):
    world, res = world_results
    n, d, b, h, seed = CASES[name]
    q, k, v, do = O.inputs(n * world, d, b, h, seed)
    if name == "bf16":
        q, k, v, do = (O.bf16_round(x) for x in (q, k, v, do))
    ref = O.lasp2_full(q, k, v, do, world, masked)
    _check(name, _cat(res, world, f"lasp2_{name}_{masked}"), ref)
    for r in range(world):  # one state all_gather per pass, no P2P (lasp2.py:211/226/260/276)
        assert res[r][f"lasp2_{name}_{masked}_ledger"] == (2, 0)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("balanced", [False, True])
def test_lasp2h_rank_programs_match_oracle(world_results, name, balanced):
    world, res = world_results
    n, d, b, h, seed = CASES[name]
    q, k, v, do = O.inputs(n * world, d, b, h, seed)
    if name == "bf16":
        q, k, v, do = (O.bf16_round(x) for x in (q, k, v, do))
    ref = O.cp_full(q, k, v, do, world, True)
    _check(name, _cat(res, world, f"cp_{name}_{balanced}"), ref)
    sends = [res[r][f"cp_{name}_{balanced}_ledger"][2] for r in range(world)]
    for r in range(world):  # K and V gathers, one dK/dV reduce_scatter (standard_sp.py:40-41, :69-75)
        assert res[r][f"cp_{name}_{balanced}_ledger"][:2] == (2, 1)
    assert (sum(sends) > 0) == balanced  # the balanced schedule pairs ranks over P2P


@pytest.mark.parametrize("name", list(CASES))
def test_lasp1_ring_rank_programs_match_oracle(world_results, name):
    world, res = world_results
    n, d, b, h, seed = CASES[name]
    q, k, v, do = O.inputs(n * world, d, b, h, seed)
    if name == "bf16":
        q, k, v, do = (O.bf16_round(x) for x in (q, k, v, do))
    ref = O.lasp2_full(q, k, v, do, world, True)
    _check(name, _cat(res, world, f"lasp1_{name}"), ref)
    # 2(W-1) P2P steps over the whole world (lasp1.py:43-107)
    assert sum(res[r][f"lasp1_{name}_ledger"][0] for r in range(world)) == 2 * (world - 1)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("masked", [True, False])
def test_peer_exchange_across_processes_matches_collective_bitwise(world_results, name, masked):
    """Same scan, same copy-first fold order: the fused peer exchange gives the all_gather
    path's bits, with one all_gather launch per exchange in the ledger."""
    world, res = world_results
    for r in range(world):
        method, fallback, launches = res[r][f"peer_{name}_{masked}_info"]
        assert fallback is None and method in ("symmetric_memory", "cuda_ipc"), (method, fallback)
        assert launches == 2
        for a, b in zip(res[r][f"peer_{name}_{masked}"], res[r][f"lasp2_{name}_{masked}"]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("masked", [True, False])
def test_peer_exchange_graph_replays_match_collective_bitwise(world_results, name, masked):
    """Three replays of a captured peer-exchange program: each replay is a fresh exchange
    (device epochs advance: 1 eager + 3 replays per state), results bitwise equal to the
    all_gather path every time."""
    world, res = world_results
    for r in range(world):
        for rep in res[r][f"peer_graph_{name}_{masked}"]:
            for a, b in zip(rep, res[r][f"lasp2_{name}_{masked}"]):
                assert np.array_equal(a, b)
        assert res[r][f"peer_graph_{name}_{masked}_epoch"] == [4, 4]  # state + state_grad exchanges
