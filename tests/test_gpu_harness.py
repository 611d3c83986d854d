"""The verify / bench harness (reference cli.py verify / bench) over the GPU
drivers: the reference's default verify grid passes in f64 (with finite
differences where the reference runs them), f32 and bf16 runs pass their
tolerances, the corrupt-gradient hook fails, and bench rows carry the
reference's ledger columns and simulated clock."""
import json

import pytest

from paper_2502_07563_b200 import harness
from paper_2502_07563_b200.harness import RunConfig

pytestmark = pytest.mark.gpu


def test_default_verify_grid_passes(tmp_path, capsys):
    out = tmp_path / "report.json"
    assert harness.main(["verify", "--out", str(out)]) == 0
    runs = json.loads(out.read_text())["runs"]
    assert len(runs) == len(harness.default_verify_grid()) and all(r["passed"] for r in runs)
    assert any(c["name"] == "backward_rel_vs_fd" for r in runs for c in r["checks"])
    assert capsys.readouterr().out.strip().endswith(f"{len(runs)}/{len(runs)} runs passed")


@pytest.mark.parametrize("method", harness.METHODS)
def test_corrupt_gradient_fails(method):
    flags = ["--pattern", "LN"] if method == "lasp2h" else []
    assert harness.main(["verify", "--method", method, "--seq-len", "16", "--chunks", "2", *flags,
                         "--corrupt-gradient"]) == 1


@pytest.mark.parametrize("precision,n,d,heads", [("f32", 256, 16, 2), ("bf16", 2048, 64, 4)])
@pytest.mark.parametrize("method", harness.METHODS)
def test_low_precision_runs_pass(method, precision, n, d, heads):
    # bf16 stacks: "NN", because an unnormalised L layer feeds the next softmax
    # logits of size ~N, where bf16 rounding flips the row maxima (an O(1)
    # change of a hard-max output, not a kernel error)
    pattern = ("LN" if precision != "bf16" else "NN") if method == "lasp2h" else ""
    cfg = RunConfig(method=method, precision=precision, seq_len=n, chunks=2, dim=d, heads=heads, pattern=pattern)
    checks, _, _ = harness.run_checks(cfg)
    assert all(c.passed for c in checks), [c.as_dict() for c in checks if not c.passed]


def test_dp_replicas_and_bench_rows(capsys):
    checks, ledger, sim = harness.run_checks(RunConfig(method="lasp2", seq_len=32, chunks=4, world=8, dim=4))
    assert all(c.passed for c in checks) and ledger["allgather_launches"] == 4
    assert harness.main(["bench", "--method", "lasp2", "--seq-len", "64", "--chunks", "4"]) == 0
    header, row = capsys.readouterr().out.strip().splitlines()
    assert header.split(",") == harness.BENCH_COLUMNS
    f = row.split(",")
    # 2 all_gathers of B*H*d^2 f64 per rank: 2 * (10 + 512/1024) simulated units
    assert f[:11] == ["lasp2", "64", "4", "4", "8", "1", "1", "true", "2", "2", str(2 * 4 * 8 * 8 * 8)]
    assert float(f[11]) == 21.0 and int(f[12]) > 0
    row = harness.bench_row(RunConfig(method="lasp1", seq_len=64, chunks=4))
    assert row[8] == 6 and row[9] == 0
