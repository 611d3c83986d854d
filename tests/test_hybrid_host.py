"""Hybrid stack (reference hybrid.py): host logic and the stack oracle against
outputs of the reference's own hybrid_iteration (tests/golden/hybrid_cases.npz,
made by tests/golden/make_golden.py hybrid). CPU only."""
import importlib.util
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

from oracle import lasp_oracle as O

_spec = importlib.util.spec_from_file_location("make_golden", Path(__file__).parent / "golden" / "make_golden.py")
_mg = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mg)
HYBRID_CASES, hybrid_key = _mg.HYBRID_CASES, _mg.hybrid_key

STACK_TOL = 1e-9  # test_hybrid.py:16


def test_model_spec_layers_and_validation():
    from paper_2502_07563_b200.hybrid import ModelSpec
    assert ModelSpec("LLLN LLLN", dim=4).layers == "LLLNLLLN"
    assert ModelSpec("L", dim=4).layers == "L"
    for bad in ("", "LXN", "   "):
        with pytest.raises(ValueError):
            ModelSpec(bad, dim=4)
    with pytest.raises(ValueError):
        ModelSpec("L", dim=0)


def test_pattern_for_ratio():
    from paper_2502_07563_b200.hybrid import pattern_for_ratio
    assert pattern_for_ratio(16, 0) == "LLLL LLLL LLLL LLLL"
    assert pattern_for_ratio(16, Fraction(1, 8)) == "LLLL LLLN LLLL LLLN"
    assert pattern_for_ratio(16, Fraction(1, 4)) == "LLLN LLLN LLLN LLLN"
    assert pattern_for_ratio(16, Fraction(1, 2)) == "LNLN LNLN LNLN LNLN"
    assert pattern_for_ratio(4, 1) == "NNNN"
    for n, r in ((16, Fraction(1, 3)), (16, 2), (16, Fraction(-1, 4)), (0, 0)):
        with pytest.raises(ValueError):
            pattern_for_ratio(n, r)


def test_layer_weights_deterministic_and_match_oracle():
    from paper_2502_07563_b200.hybrid import ModelSpec, layer_weights
    spec = ModelSpec("LN", dim=4, seed=3)
    ws = layer_weights(spec)
    assert len(ws) == 2 and all(w.shape == (4, 4) for t in ws for w in t)
    ref = O.stack_weights("LN", 4, 3)
    assert all(np.array_equal(a, b) for ta, tb in zip(ws, ref) for a, b in zip(ta, tb))
    assert not np.array_equal(ws[0][0], ws[1][0])
    assert layer_weights(ModelSpec("L", dim=4, seed=7))[0][0][0, 0] == 0.3980089845330995


@pytest.mark.parametrize("case", HYBRID_CASES, ids=lambda c: hybrid_key(*c))
def test_stack_oracle_matches_reference(hybrid_golden, case):
    pattern, n, d, t, b, h, seed, causal = case
    x = O.gen_slots(seed, b, h, n, d, "x")
    dy = O.gen_slots(seed, b, h, n, d, "dy")
    out, dx, dw, _ = O.stack_iteration(pattern, x, dy, causal, seed=seed, bc=8)
    key = hybrid_key(*case)
    assert O.relative_error(out, hybrid_golden[key + "_out"]) <= STACK_TOL
    assert O.relative_error(dx, hybrid_golden[key + "_dx"]) <= STACK_TOL
    assert O.relative_error(np.stack([np.stack(w) for w in dw]), hybrid_golden[key + "_dw"]) <= STACK_TOL
    layers = pattern.replace(" ", "")
    assert hybrid_golden[key + "_ledger"][0] == 2 * layers.count("L") + 3 * layers.count("N")
