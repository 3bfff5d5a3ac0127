"""Drop-in API surface of paper_2508_02932_b200.lorapack vs the reference
(names, error substrings, offsets, round trip) -- runs on CPU (no compute)."""

from pathlib import Path

import numpy as np
import pytest

import paper_2508_02932_b200.lorapack as L

REF_ALL = ["AdapterWeights", "PackedAdapters", "GradCheckReport", "pack_adapters", "unpack_adapters",
           "adapter_forward", "adapter_backward", "packed_forward", "packed_backward", "grad_check"]


def random_pack(rng, n_adapters, d, k, max_rank=8, max_tokens=6):
    # same generator as pkg/tests/test_lorapack.py:16-25
    adapters, inputs = [], []
    for _ in range(n_adapters):
        r = int(rng.integers(1, max_rank + 1))
        tokens = int(rng.integers(1, max_tokens + 1))
        adapters.append(L.AdapterWeights(down=rng.standard_normal((d, r)), up=rng.standard_normal((r, k)),
                                         alpha=float(rng.uniform(0.1, 2.0))))
        inputs.append(rng.standard_normal((tokens, d)))
    return adapters, inputs, L.pack_adapters(adapters, inputs)


def test_public_names():
    assert L.__all__ == REF_ALL
    import paper_2508_02932_b200 as pkg
    for name in REF_ALL:
        assert getattr(pkg, name) is getattr(L, name)


def test_offsets_and_round_trip():
    rng = np.random.default_rng(1)
    adapters = [L.AdapterWeights(rng.standard_normal((4, 8)), rng.standard_normal((8, 5)), 1.0),
                L.AdapterWeights(rng.standard_normal((4, 16)), rng.standard_normal((16, 5)), 1.0)]
    packed = L.pack_adapters(adapters, [rng.standard_normal((3, 4)), rng.standard_normal((2, 4))])
    assert packed.rank_offsets == (0, 8, 24)
    assert packed.row_offsets == (0, 3, 5)
    rng = np.random.default_rng(2)
    adapters, inputs, packed = random_pack(rng, 4, d=6, k=5)
    back_adapters, back_inputs = L.unpack_adapters(packed)
    for orig, back in zip(adapters, back_adapters):
        np.testing.assert_array_equal(orig.down, back.down)
        np.testing.assert_array_equal(orig.up, back.up)
        assert orig.alpha == back.alpha
    for orig, back in zip(inputs, back_inputs):
        np.testing.assert_array_equal(orig, back)


def test_error_messages_match_reference():
    rng = np.random.default_rng(3)
    a = L.AdapterWeights(rng.standard_normal((4, 2)), rng.standard_normal((2, 5)), 1.0)
    b = L.AdapterWeights(rng.standard_normal((6, 2)), rng.standard_normal((2, 5)), 1.0)
    with pytest.raises(ValueError, match="adapter 1"):
        L.pack_adapters([a, b], [rng.standard_normal((2, 4))] * 2)
    with pytest.raises(ValueError, match="rank mismatch"):
        L.AdapterWeights(rng.standard_normal((4, 2)), rng.standard_normal((3, 5)), 1.0)
    with pytest.raises(ValueError, match="nothing to pack"):
        L.pack_adapters([], [])
    with pytest.raises(ValueError, match="1 adapters but 2 inputs"):
        L.pack_adapters([a], [rng.standard_normal((2, 4))] * 2)
    with pytest.raises(ValueError, match="input 0 must be"):
        L.pack_adapters([a], [rng.standard_normal((2, 3))])
    _, _, packed = random_pack(np.random.default_rng(8), 1, d=4, k=3)
    with pytest.raises(ValueError, match="base weight"):
        L.packed_forward(packed, rng.standard_normal((3, 3)))
    _, inputs, packed = random_pack(np.random.default_rng(12), 2, d=4, k=3)
    bad = [np.zeros((inputs[0].shape[0], 3)), np.zeros((inputs[1].shape[0] + 1, 3))]
    with pytest.raises(ValueError, match="upstream 1"):
        L.packed_backward(packed, rng.standard_normal((4, 3)), bad)


def test_packed_invariants_rejected():
    with pytest.raises(ValueError, match="strictly increasing"):
        L.PackedAdapters(np.zeros((2, 2)), np.zeros((2, 3)), np.zeros((1, 2)), (1.0, 1.0), (0, 2, 2), (0, 1, 1))
    with pytest.raises(ValueError, match="partition the packed sequence"):
        L.PackedAdapters(np.zeros((2, 2)), np.zeros((2, 3)), np.zeros((2, 2)), (1.0,), (0, 2), (0, 1))


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    _, _, packed = random_pack(np.random.default_rng(4), 2, d=5, k=4)
    with pytest.raises(RuntimeError):
        L.packed_forward(packed, np.zeros((5, 4)))


_REF_TESTS = Path("/root/reference/pkg/tests/test_lorapack.py")


@pytest.mark.skipif(not _REF_TESTS.exists(), reason="reference checkout not present")
def test_reference_packing_tests_verbatim():
    """The reference's own test file run against this drop-in through the module alias
    (tests/_lorasweep_alias.py): TestPacking (offset goldens, round trip, shape errors --
    the bit-exact indexing contract) and the argument-validation tests that fail before
    any device work.  Its float64 numeric tests (1e-12 / 1e-10 bounds) are exercised at
    the bf16 tier in tests/test_gpu_lorapack.py instead."""
    import os
    import subprocess
    import sys

    root = Path(__file__).resolve().parent.parent
    sel = ("TestPacking or test_wrong_base_shape or test_upstream_shape_checked")
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", PYTHONPATH=f"{root}:{root / 'tests'}")
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "_lorasweep_alias", "-p", "no:cacheprovider", "-q",
                        "-k", sel, str(_REF_TESTS)], cwd="/tmp", env=env, capture_output=True, text=True, timeout=600)
    tail = r.stdout[-2000:]
    assert r.returncode == 0, tail
    assert "6 passed" in tail, tail
