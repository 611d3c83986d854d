"""Host side of the verify / bench / cost-table harness (reference cli.py):
the cost table is byte-identical to the reference CLI's default table
(tests/golden/costmodel_default.csv, made by make_golden.py costmodel), the
CSV columns are the reference's, and configuration errors are UsageErrors
(exit code 2) in the same cases."""
from pathlib import Path

import pytest

from paper_2502_07563_b200 import harness
from paper_2502_07563_b200.harness import RunConfig, UsageError

GOLDEN_DIR = Path(__file__).parent / "golden"


def test_cost_table_matches_reference(tmp_path):
    out = tmp_path / "cost.csv"
    assert harness.main(["costmodel", "--out", str(out)]) == 0
    assert out.read_text() == (GOLDEN_DIR / "costmodel_default.csv").read_text()


def test_cost_flags_and_errors(tmp_path, capsys):
    assert harness.main(["costmodel", "--method", "lasp2", "--world", "8", "--heads", "16", "--dim", "128",
                         "--element-bytes", "2"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0].split(",") == harness.COST_COLUMNS
    assert lines[1] == "lasp2,8,8,1,16,128,2,1,2,524288,262144,1048576"
    assert harness.main(["costmodel", "--world", "8", "--chunks", "3"]) == 2


def test_columns_are_the_references():
    assert harness.BENCH_COLUMNS == ["method", "N", "T", "W", "d", "H", "B", "masked", "steps", "launches",
                                     "bytes", "simulated_time", "wall_time_ns"]


@pytest.mark.parametrize("kwargs", [
    {"method": "oracle"}, {"method": "ring"}, {"precision": "f16"}, {"seq_len": 0}, {"seq_len": 10, "chunks": 4},
    {"world": 6, "chunks": 4}, {"method": "lasp2h"}, {"pattern": "LN"}, {"latency_per_byte": -1.0},
])
def test_run_config_rejects(kwargs):
    with pytest.raises(UsageError):
        RunConfig(**kwargs)


def test_run_config_defaults_and_hash():
    cfg = RunConfig()
    assert cfg.world == cfg.chunks == 4 and cfg.element_bytes == 8
    assert RunConfig(precision="bf16").element_bytes == 2
    assert cfg.config_hash() == RunConfig().config_hash() != RunConfig(seed=1).config_hash()
    wc = RunConfig(world=8, chunks=4, precision="f32").world_config()
    assert (wc.world_size, wc.sp_size, wc.element_bytes) == (8, 4, 4)


def test_config_and_grid_files(tmp_path):
    conf = tmp_path / "run.conf"
    conf.write_text("# base\nmethod = lasp1\nseq-len = 32\n")
    grid = tmp_path / "grid.conf"
    grid.write_text("chunks = 1, 2, 4\nmasked = true, false\n")
    parser = harness.build_parser()
    args = parser.parse_args(["bench", "--config", str(conf), "--grid", str(grid), "--dim", "4"])
    runs = harness._expand(args, harness._RUN_KEYS, lambda: [{}])
    assert len(runs) == 6
    assert all(r["method"] == "lasp1" and r["seq_len"] == 32 and r["dim"] == 4 for r in runs)
    assert {(r["chunks"], r["masked"]) for r in runs} == {(t, m) for t in (1, 2, 4) for m in (True, False)}
    bad = tmp_path / "bad.conf"
    bad.write_text("colour = red\n")
    with pytest.raises(UsageError):
        harness._config_file(str(bad), harness._RUN_KEYS)
    dup = tmp_path / "dup.conf"
    dup.write_text("chunks = 1\nchunks = 2\n")
    with pytest.raises(UsageError):
        harness._grid_file(str(dup), harness._RUN_KEYS)


def test_default_verify_grid_shape():
    grid = harness.default_verify_grid()
    assert len(grid) == 4 * 3 * 4 * 2 * 2  # every (n, t) divides
    assert all(g["pattern"] == ("LN" if g["method"] == "lasp2h" else "") for g in grid)
    for g in grid:
        RunConfig(**g)


def test_bad_flags_exit_2():
    assert harness.main(["verify", "--method", "lasp2", "--seq-len", "ten"]) == 2
    assert harness.main(["nonsense"]) == 2
