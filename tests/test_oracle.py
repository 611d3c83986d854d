"""The oracle (tests' checker) against the reference's own goldens and fixtures.

Fixtures in tests/golden/reference_cases.npz were produced by running the
reference implementation (tests/golden/make_golden.py); the datagen goldens are
the reference test suite's constants (pkg/tests/test_datagen.py:9-17, :82).
"""
import numpy as np
import pytest

from oracle import lasp_oracle as O

GOLDEN_SEED0_2X2 = np.array([[0.6430912012993306, -0.9298324997834873],
                             [-0.22244924825266255, -0.15583515821469263]])
GOLDEN_SEED1_1X4 = np.array([[0.7941861682853886, -0.10429277713750951, -0.8561598952806655, -0.5483075560653927]])
GOLDEN_SEED0_TAG_Q = np.array([[0.37493450945250384, -0.29778935369585713]])

LASP_CASES = [(8, 4, 1, 1, 1, 0), (8, 4, 2, 1, 1, 0), (16, 8, 4, 1, 1, 0), (16, 4, 8, 1, 1, 0),
              (64, 16, 4, 1, 1, 0), (256, 16, 8, 1, 1, 0), (256, 4, 2, 1, 1, 0), (8, 4, 4, 2, 3, 5),
              (256, 32, 4, 1, 2, 7)]
CP_CASES = [(8, 4, 2, 1, 1, 0), (16, 8, 4, 1, 1, 0), (16, 4, 2, 1, 1, 0), (8, 4, 4, 2, 2, 3), (256, 32, 4, 1, 2, 1)]


def test_datagen_goldens():
    assert np.array_equal(O.gen_data(0, 2, 2), GOLDEN_SEED0_2X2)
    assert np.array_equal(O.gen_data(1, 1, 4), GOLDEN_SEED1_1X4)
    assert np.array_equal(O.gen_data(0, 1, 2, tag="q"), GOLDEN_SEED0_TAG_Q)
    w = O.gen_data(7, 4, 4, tag="wq/layer0") / np.sqrt(4.0)
    assert w[0, 0] == 0.3980089845330995


def test_product_datagen_matches_oracle():
    from paper_2502_07563_b200 import datagen
    assert np.array_equal(datagen.gen_data(0, 2, 2), GOLDEN_SEED0_2X2)
    assert np.array_equal(datagen.gen_slots(3, 2, 3, 4, 5, "q"), O.gen_slots(3, 2, 3, 4, 5, "q"))
    assert datagen.projection_weight(7, 0, "q", 4)[0, 0] == 0.3980089845330995


def test_hand_examples():
    q, k, v = np.array([[1.0], [1.0]]), np.array([[1.0], [2.0]]), np.array([[1.0], [1.0]])
    assert np.array_equal(O.causal_linear_forward(q, k, v), [[1.0], [3.0]])
    q, k, v = np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]]), np.array([[5.0], [6.0]])
    assert np.array_equal(O.linear_attn_serial(q, k, v, True), [[15.0], [78.0]])
    assert np.array_equal(O.linear_attn_serial(q, k, v, False), [[39.0], [78.0]])


def test_fold_order_contract():
    s = [np.array([-0.0, 1.0]), np.array([-0.0, 2.0]), np.array([-0.0, 4.0])]
    p = O.prefix_sum_states(s, 2)
    assert np.signbit(p[0]) and p[1] == 3.0  # copy-first keeps -0.0 (numerics.py:6-8)
    assert np.array_equal(O.prefix_sum_states(s, 0), [0.0, 0.0])
    assert np.array_equal(O.suffix_sum_states(s, 3), [0.0, 0.0])
    assert O.suffix_sum_states(s, 1)[1] == 6.0 and np.signbit(O.suffix_sum_states(s, 1)[0])
    assert O.sum_states(s)[1] == 7.0


@pytest.mark.parametrize("masked", [True, False])
@pytest.mark.parametrize("case", LASP_CASES)
def test_oracle_matches_reference_lasp2(golden, case, masked):
    n, d, t, b, h, seed = case
    q, k, v, do = O.inputs(n, d, b, h, seed)
    out, dq, dk, dv = O.lasp2_full(q, k, v, do, t, masked, bc=4)
    key = f"lasp2_{'m' if masked else 'u'}_{n}_{d}_{t}_{b}_{h}_{seed}"
    assert np.max(np.abs(out - golden[key + "_out"])) <= 1e-10
    for name, g in (("dq", dq), ("dk", dk), ("dv", dv)):
        assert O.relative_error(g, golden[f"{key}_{name}"]) <= 1e-12


def test_oracle_matches_reference_cfg1(golden):
    rows = golden["cfg1_rows"]
    q, k, v, do = O.inputs(4096, 64, 1, 4, 0)
    got = dict(zip(("out", "dq", "dk", "dv"), O.lasp2_full(q, k, v, do, 2, True, bc=256)))
    for name, arr in got.items():
        ref = golden[f"cfg1_{name}_rows"]
        assert O.normalized_error(arr[:, :, rows, :], ref) <= 1e-12, name
        s = golden[f"cfg1_{name}_sum"]
        assert abs(arr.sum() - s[0]) <= 1e-9 * s[1] ** 0.5 * 64
        assert abs(np.abs(arr).max() - s[2]) <= 1e-9 * s[2]


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("case", CP_CASES)
def test_oracle_matches_reference_cp(golden, case, causal):
    n, d, t, b, h, seed = case
    q, k, v, do = O.inputs(n, d, b, h, seed)
    out, dq, dk, dv = O.cp_full(q, k, v, do, t, causal)
    key = f"cp_{'c' if causal else 'n'}_{n}_{d}_{t}_{b}_{h}_{seed}"
    assert np.max(np.abs(out - golden[key + "_out"])) <= 1e-12
    for name, g in (("dq", dq), ("dk", dk), ("dv", dv)):
        assert O.relative_error(g, golden[f"{key}_{name}"]) <= 1e-10


def test_blocked_intra_equals_per_token():
    q, k, v, do = O.inputs(40, 8, 1, 1, 7)
    ref = O.causal_linear_forward(q[0, 0], k[0, 0], v[0, 0])
    for bc in (1, 3, 16, 64):
        assert np.max(np.abs(O.intra_forward_blocked(q, k, v, bc)[0, 0] - ref)) <= 1e-12
    rq, rk, rv = O.linear_attn_serial_backward(q[0, 0], k[0, 0], v[0, 0], do[0, 0], True)
    dq, dk, dv = O.intra_backward_blocked(q, k, v, do, 7)
    for g, r in ((dq, rq), (dk, rk), (dv, rv)):
        assert O.relative_error(g[0, 0], r) <= 1e-12


def test_bf16_round_matches_torch():
    import torch
    x = O.gen_data(11, 64, 64) * 300.0
    want = torch.from_numpy(x).float().bfloat16().double().numpy()
    assert np.array_equal(O.bf16_round(x), want)


def test_c_datagen_matches_numpy_restatement():
    """oracle/datagen.c (bench.py's full-size CPU inputs) is bit-exact with gen_data."""
    import numpy as np

    lib = O._c_datagen()
    if lib is None:
        pytest.skip("oracle/liboracle_datagen.so not built (make -C oracle)")
    saved = list(O._CGEN)
    for dt in (np.float64, np.float32):
        O._CGEN[:] = [lib]
        fast = O.gen_data(7, 1024, 96, "v/b0/h3", dt)
        O._CGEN[:] = [None]
        slow = O.gen_data(7, 1024, 96, "v/b0/h3", dt)
        O._CGEN[:] = saved
        assert fast.dtype == slow.dtype and np.array_equal(fast, slow)
