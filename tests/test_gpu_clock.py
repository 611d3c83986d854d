"""The threads-as-ranks world's simulated clock (reference comm.py:7-12:
only communication moves a rank's clock; a P2P message arrives at the send
clock plus latency_per_launch + bytes * latency_per_byte; a collective
completes for everyone at the latest issue clock plus the same cost), pinned
to WorldRun.simulated_time of the reference's own drivers
(tests/golden/clock_cases.json, made by tests/golden/make_golden.py clock)
together with the ledger's step and byte counts, and the reference's
acceptance criterion 9 (test_acceptance.py:237-252)."""
import json
from pathlib import Path

import pytest
import torch

from oracle import lasp_oracle as O
from paper_2502_07563_b200 import comm
from paper_2502_07563_b200.hybrid import ModelSpec, hybrid_iteration
from paper_2502_07563_b200.lasp1 import lasp1_iteration
from paper_2502_07563_b200.lasp2 import ChunkedSequence, lasp2_iteration
from paper_2502_07563_b200.standard_sp import cp_iteration

pytestmark = pytest.mark.gpu

CASES = json.loads((Path(__file__).parent / "golden" / "clock_cases.json").read_text())


@pytest.mark.parametrize("row", CASES, ids=lambda r: "_".join(str(x) for x in r["case"][:5]))
def test_simulated_time_matches_reference(row):
    method, n, d, t, world, b, h, masked, pattern, lat_l, lat_b = row["case"]
    cfg = comm.WorldConfig(world_size=world, sp_size=t, element_bytes=8,
                           latency_per_launch=lat_l, latency_per_byte=lat_b)
    if method == "hybrid":
        spec = ModelSpec(pattern, dim=d, heads=h, batch=b, seed=0)
        run = hybrid_iteration(spec, O.gen_slots(0, b, h, n, d, "x"), O.gen_slots(0, b, h, n, d, "dy"),
                               t, masked, cfg).run
    else:
        q, k, v, do = O.inputs(n, d, b, h)
        seq = ChunkedSequence(q, k, v, t)
        if method == "lasp2_overlap":
            run = lasp2_iteration(seq, do, masked, cfg, overlap=True).run
        else:
            driver = {"lasp2": lasp2_iteration, "lasp1": lasp1_iteration, "cp": cp_iteration}[method]
            run = driver(seq, do, masked, cfg).run
    assert run.simulated_time == row["simulated_time"]
    assert run.stats.communication_steps == row["communication_steps"]
    assert run.stats.bytes_sent == row["bytes_sent"]


def test_criterion_9_simulated_latency_ordering():
    for world in (4, 8):
        q, k, v, do = O.inputs(8 * world, 4)
        seq = ChunkedSequence(q, k, v, world)
        ring, gather = lasp1_iteration(seq, do, True), lasp2_iteration(seq, do, True)
        assert gather.run.simulated_time < ring.run.simulated_time, world
        free = comm.WorldConfig(world, latency_per_byte=0.0)
        ratio = (lasp1_iteration(seq, do, True, free).run.simulated_time
                 / lasp2_iteration(seq, do, True, free).run.simulated_time)
        assert ratio >= 0.5 * (world - 1), (world, ratio)


def test_barrier_aligns_clocks_without_accounting():
    def program(ctx):
        if ctx.rank == 1:
            ctx.send(0, torch.zeros(4, device="cuda"))
        if ctx.rank == 0:
            ctx.recv(1)
        ctx.barrier()
        return ctx.clock

    cfg = comm.WorldConfig(2, latency_per_launch=5.0, latency_per_byte=0.0)
    run = comm.world_spawn(cfg, program)
    assert run.results == [5.0, 5.0]
    assert run.stats.communication_steps == 1 and run.stats.allgather_launches == 0
