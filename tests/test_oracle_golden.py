"""The oracle (oracle/lorapack_oracle.py) is pinned against the REAL reference:
golden vectors from oracle/gen_golden.py and the known-answer values of the
reference's own tests (pkg/tests/test_lorapack.py)."""

import numpy as np
import pytest

from oracle import lorapack_oracle as O
from tests.conftest import split_cols, split_rows


def test_golden_cases_match_oracle(golden_cases):
    assert len(golden_cases) >= 17
    for name, c in golden_cases:
        ro, so = c["rank_offsets"], c["row_offsets"]
        downs = split_cols(c["down_block"], ro)
        ups = [c["up_block"][ro[i]:ro[i + 1]] for i in range(len(ro) - 1)]
        inputs = split_rows(c["inputs"], so)
        p = O.pack(downs, ups, c["alphas"], inputs)
        assert p["rank_offsets"] == ro, name
        assert p["row_offsets"] == so, name
        ys = O.packed_forward(p, c["w"])
        np.testing.assert_allclose(np.concatenate(ys, axis=0), c["y"], rtol=0, atol=1e-12, err_msg=name)
        dd, du, dx = O.packed_backward(p, c["w"], split_rows(c["upstream"], so))
        np.testing.assert_allclose(np.concatenate(dd, axis=1), c["d_down"], atol=1e-10, err_msg=name)
        np.testing.assert_allclose(np.concatenate(du, axis=0), c["d_up"], atol=1e-10, err_msg=name)
        np.testing.assert_allclose(np.concatenate(dx, axis=0), c["d_input"], atol=1e-10, err_msg=name)


def test_known_answers_from_reference_tests():
    # pkg/tests/test_lorapack.py:29-46 -- offset goldens
    rng = np.random.default_rng(1)
    p = O.pack([rng.standard_normal((4, 8)), rng.standard_normal((4, 16))],
               [rng.standard_normal((8, 5)), rng.standard_normal((16, 5))], [1.0, 1.0],
               [rng.standard_normal((3, 4)), rng.standard_normal((2, 4))])
    assert p["rank_offsets"] == (0, 8, 24)
    assert p["row_offsets"] == (0, 3, 5)
    assert O.prefix_offsets([3]) == (0, 3)
    # :70-74 forward scalar 2*3 + 0.5*(2*1)*1 = 7
    p = O.pack([np.array([[1.0]])], [np.array([[1.0]])], [0.5], [np.array([[2.0]])])
    assert O.packed_forward(p, np.array([[3.0]]))[0][0, 0] == pytest.approx(7.0)
    # :129-136 backward scalar dB=1, dA=1, dx=3.5
    dd, du, dx = O.packed_backward(p, np.array([[3.0]]), [np.array([[1.0]])])
    assert du[0][0, 0] == pytest.approx(1.0)
    assert dd[0][0, 0] == pytest.approx(1.0)
    assert dx[0][0, 0] == pytest.approx(3.5)


def test_packed_equals_sequential_oracle():
    # reference crit. 1 shape family (pkg/tests/test_acceptance.py:165-201), smaller count
    rng = np.random.default_rng(101)
    for _ in range(50):
        n, d, k = int(rng.integers(1, 9)), int(rng.integers(2, 33)), int(rng.integers(2, 33))
        downs, ups, al, xs, dys = [], [], [], [], []
        for _ in range(n):
            r, t = int(rng.integers(1, 17)), int(rng.integers(0, 9))
            downs.append(rng.standard_normal((d, r)))
            ups.append(rng.standard_normal((r, k)))
            al.append(float(rng.uniform(0.1, 2.0)))
            xs.append(rng.standard_normal((t, d)))
            dys.append(rng.standard_normal((t, k)))
        w = rng.standard_normal((d, k))
        p = O.pack(downs, ups, al, xs)
        ys = O.packed_forward(p, w)
        dd, du, dx = O.packed_backward(p, w, dys)
        for i in range(n):
            np.testing.assert_allclose(ys[i], O.single_forward(downs[i], ups[i], al[i], xs[i], w), atol=1e-12)
            rd, ru, rx = O.single_backward(downs[i], ups[i], al[i], xs[i], w, dys[i])
            np.testing.assert_allclose(dd[i], rd, atol=1e-10)
            np.testing.assert_allclose(du[i], ru, atol=1e-10)
            np.testing.assert_allclose(dx[i], rx, atol=1e-10)


def test_token_adapter_ids():
    ids = O.token_adapter_ids((0, 3, 3, 7))
    assert ids.tolist() == [0, 0, 0, 2, 2, 2, 2]
