"""Drop-in list-based folds (paper_2502_07563_b200.numerics, reference numerics.py:60-121):
host-side validation here, bitwise agreement with the oracle's copy-first loops on the GPU."""
import numpy as np
import pytest
import torch

from oracle import lasp_oracle as O
from paper_2502_07563_b200 import numerics as N


def test_validation_matches_reference_errors():
    with pytest.raises(ValueError, match="non-empty"):
        N.prefix_sum_states([], 0)
    a, b = torch.zeros(2, 2, dtype=torch.float64), torch.zeros(3, 2, dtype=torch.float64)
    with pytest.raises(ValueError, match="state 1 has shape"):
        N.sum_states([a, b])
    with pytest.raises(ValueError, match="upto=3 outside"):
        N.prefix_sum_states([a, a], 3)
    with pytest.raises(ValueError, match="start=-1 outside"):
        N.suffix_sum_states([a, a], -1)
    with pytest.raises(ValueError, match="float32 or float64"):
        N.sum_states([a.to(torch.bfloat16)] * 2)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_folds_bitwise_equal_oracle(dtype):
    rng = np.random.default_rng(3)
    states = [rng.standard_normal((2, 4, 8, 8)).astype(dtype) for _ in range(5)]
    states[0][0, 0, 0, 0] = -0.0  # copy-first seeding keeps -0.0 (numerics.py:6-8)
    for s in states[1:]:
        s[0, 0, 0, 0] = -0.0
    dev = [torch.from_numpy(s).cuda() for s in states]
    for upto in range(6):
        got = N.prefix_sum_states(dev, upto).cpu().numpy()
        assert np.array_equal(got, O.prefix_sum_states(states, upto))
        assert np.array_equal(np.signbit(got), np.signbit(O.prefix_sum_states(states, upto)))
    for start in range(6):
        got = N.suffix_sum_states(torch.stack(dev), start).cpu().numpy()
        assert np.array_equal(got, O.suffix_sum_states(states, start))
    assert np.array_equal(N.sum_states(dev).cpu().numpy(), O.sum_states(states))
