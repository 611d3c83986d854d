"""LASP-1 ring baseline (reference lasp1.py): the oracle against outputs of the
reference's own lasp1_iteration (tests/golden/lasp1_cases.npz, made by
tests/golden/make_golden.py lasp1). CPU only."""
import importlib.util
from pathlib import Path

import numpy as np
import pytest

from oracle import lasp_oracle as O

_spec = importlib.util.spec_from_file_location("make_golden", Path(__file__).parent / "golden" / "make_golden.py")
_mg = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mg)
LASP1_CASES = _mg.LASP1_CASES


@pytest.mark.parametrize("masked", [True, False])
@pytest.mark.parametrize("case", LASP1_CASES)
def test_oracle_matches_reference_ring(lasp1_golden, case, masked):
    n, d, t, b, h, seed = case
    q, k, v, do = O.inputs(n, d, b, h, seed)
    key = f"l1_{'m' if masked else 'u'}_{n}_{d}_{t}_{b}_{h}_{seed}"
    if masked:  # the ring's masked results are the all_gather method's (lasp1.py:6-9)
        got = O.lasp2_full(q, k, v, do, t, True, bc=4)
    else:
        got = O.lasp1_nomask_full(q, k, v, do, t)
    for g, nm in zip(got, ("out", "dq", "dk", "dv")):
        assert O.relative_error(g, lasp1_golden[f"{key}_{nm}"]) <= 1e-10, nm
    # final ring state = full sum of the chunk states (test_lasp1.py:142-148)
    c = n // t
    states = [np.swapaxes(k[:, :, i * c:(i + 1) * c], -1, -2) @ v[:, :, i * c:(i + 1) * c] for i in range(t)]
    assert O.relative_error(O.sum_states(states), lasp1_golden[key + "_through"]) <= 1e-12
    sends, ag, steps, nbytes = lasp1_golden[key + "_ledger"]
    assert sends == steps == 2 * (t - 1) and ag == 0
    assert nbytes == 2 * (t - 1) * b * h * d * d * 8
