"""GPU parity of the drop-in packed-LoRA API vs the reference (golden vectors made
by the real lorasweep) and vs the oracle, at the bf16 tier stated in DESIGN.md:
    relative Frobenius error <= 1e-2  and  max|err| / max|ref| <= 2e-2
Indexing is bit-exact; exact-zero cases are exact."""

import numpy as np
import pytest

import paper_2508_02932_b200.lorapack as L
from oracle import lorapack_oracle as O
from tests.conftest import split_cols, split_rows

pytestmark = pytest.mark.gpu

REL_FROB = 1e-2
MAX_REL = 2e-2


def close(got, ref, what):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, what
    if ref.size == 0 or np.max(np.abs(ref)) == 0:
        assert np.max(np.abs(got), initial=0.0) < 1e-6, what
        return
    rf = O.rel_frobenius(got, ref)
    mr = O.max_abs_over_max_ref(got, ref)
    assert rf <= REL_FROB and mr <= MAX_REL, f"{what}: rel_frob={rf:.3e} max_rel={mr:.3e}"


def _bf(a):
    import torch
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def emulate_bf16(c):
    """The oracle's algebra with the GPU path's rounding points: bf16 operands, fp32+
    accumulation, Hs = bf16(alpha X A) and dH = bf16(alpha dY B^T) stored in bf16."""
    ro, so = c["rank_offsets"], c["row_offsets"]
    X, W, dY = _bf(c["inputs"]), _bf(c["w"]), _bf(c["upstream"])
    A_all, B_all = _bf(c["down_block"]), _bf(c["up_block"])
    dd, du = [], []
    for i, al in enumerate(c["alphas"]):
        rows, cols = slice(so[i], so[i + 1]), slice(ro[i], ro[i + 1])
        A, B = A_all[:, cols], B_all[cols, :]
        hs = _bf(al * (X[rows] @ A))
        dh = _bf(al * (dY[rows] @ B.T))
        dd.append(X[rows].T @ dh)
        du.append(hs.T @ dY[rows])
    return dd, du


def _pack_case(c):
    ro, so = c["rank_offsets"], c["row_offsets"]
    downs = split_cols(c["down_block"], ro)
    ups = [c["up_block"][ro[i]:ro[i + 1]] for i in range(len(ro) - 1)]
    adapters = [L.AdapterWeights(a, b, al) for a, b, al in zip(downs, ups, c["alphas"])]
    return adapters, split_rows(c["inputs"], so)


def test_golden_forward_backward(golden_cases):
    for name, c in golden_cases:
        adapters, inputs = _pack_case(c)
        packed = L.pack_adapters(adapters, inputs)
        assert packed.rank_offsets == c["rank_offsets"] and packed.row_offsets == c["row_offsets"]
        ys = L.packed_forward(packed, c["w"])
        close(np.concatenate(ys, axis=0), c["y"], f"{name} y")
        dd, du, dx = L.packed_backward(packed, c["w"], split_rows(c["upstream"], c["row_offsets"]))
        close(np.concatenate(dd, axis=1), c["d_down"], f"{name} d_down")
        close(np.concatenate(du, axis=0), c["d_up"], f"{name} d_up")
        close(np.concatenate(dx, axis=0), c["d_input"], f"{name} d_input")
        # per adapter (a tiny segment must not hide inside the aggregate): against the
        # oracle algebra evaluated at the GPU path's bf16 rounding points, fp32-accurate
        edd, edu = emulate_bf16(c)
        for i in range(len(adapters)):
            for got, ref, what in ((dd[i], edd[i], "d_down"), (du[i], edu[i], "d_up")):
                if np.max(np.abs(ref), initial=0.0) > 0:
                    assert O.rel_frobenius(got, ref) < 1e-4, f"{name} {what}[{i}]"


def test_scalar_cases():
    # reference pkg/tests/test_lorapack.py:70-74, 129-136 (exact in bf16)
    a = L.AdapterWeights(down=np.array([[1.0]]), up=np.array([[1.0]]), alpha=0.5)
    packed = L.pack_adapters([a], [np.array([[2.0]])])
    assert L.packed_forward(packed, np.array([[3.0]]))[0][0, 0] == pytest.approx(7.0)
    dd, du, dx = L.packed_backward(packed, np.array([[3.0]]), [np.array([[1.0]])])
    assert du[0][0, 0] == pytest.approx(1.0)
    assert dd[0][0, 0] == pytest.approx(1.0)
    assert dx[0][0, 0] == pytest.approx(3.5)


def random_pack(rng, n, d, k, max_rank=8, max_tokens=6):
    adapters, inputs = [], []
    for _ in range(n):
        r = int(rng.integers(1, max_rank + 1))
        t = int(rng.integers(1, max_tokens + 1))
        adapters.append(L.AdapterWeights(rng.standard_normal((d, r)), rng.standard_normal((r, k)),
                                         float(rng.uniform(0.1, 2.0))))
        inputs.append(rng.standard_normal((t, d)))
    return adapters, inputs, L.pack_adapters(adapters, inputs)


def test_zero_alpha_and_zero_up_vanish():
    rng = np.random.default_rng(4)
    adapters, inputs, _ = random_pack(rng, 3, d=5, k=4)
    w = rng.standard_normal((5, 4))
    for mk in (lambda a: L.AdapterWeights(a.down, a.up, 0.0),
               lambda a: L.AdapterWeights(a.down, np.zeros_like(a.up), a.alpha)):
        packed = L.pack_adapters([mk(a) for a in adapters], inputs)
        base = L.packed_forward(packed, w)
        for y, x in zip(base, inputs):
            close(y, x @ w, "zero lora")
    # alpha = 0 -> dA = dB = 0 exactly
    a = L.AdapterWeights(rng.standard_normal((5, 2)), rng.standard_normal((2, 4)), 0.0)
    x = rng.standard_normal((3, 5))
    dd, du, dx = L.packed_backward(L.pack_adapters([a], [x]), w, [rng.standard_normal((3, 4))])
    assert not np.any(dd[0]) and not np.any(du[0])


def test_zero_upstream_exact_zeros():
    rng = np.random.default_rng(11)
    adapters, inputs, packed = random_pack(rng, 2, d=4, k=3)
    zeros = [np.zeros((x.shape[0], 3)) for x in inputs]
    dd, du, dx = L.packed_backward(packed, rng.standard_normal((4, 3)), zeros)
    for g in dd + du + dx:
        assert not np.any(g)


def test_packed_equals_sequential():
    # reference pkg/tests/test_lorapack.py:94-104 / 150-164 at the bf16 tier
    rng = np.random.default_rng(6)
    for _ in range(10):
        n, d, k = int(rng.integers(1, 8)), int(rng.integers(2, 12)), int(rng.integers(2, 12))
        adapters, inputs, packed = random_pack(rng, n, d, k)
        w = rng.standard_normal((d, k))
        ups = [rng.standard_normal((x.shape[0], k)) for x in inputs]
        outs = L.packed_forward(packed, w)
        dd, du, dx = L.packed_backward(packed, w, ups)
        for i, (a, x, dy) in enumerate(zip(adapters, inputs, ups)):
            close(outs[i], L.adapter_forward(a, x, w), "fwd packed vs single")
            rd, ru, rx = L.adapter_backward(a, x, w, dy)
            close(dd[i], rd, "dA packed vs single")
            close(du[i], ru, "dB packed vs single")
            close(dx[i], rx, "dX packed vs single")
            # and both vs the fp64 oracle
            close(outs[i], O.single_forward(a.down, a.up, a.alpha, x, w), "fwd vs oracle")


def test_empty_segment_and_big_rank():
    rng = np.random.default_rng(21)
    d, k = 72, 40
    specs = [(3, 5), (130, 0), (64, 140), (1, 129)]
    adapters = [L.AdapterWeights(rng.standard_normal((d, r)) / 8, rng.standard_normal((r, k)) / 8, 0.7)
                for r, _ in specs]
    inputs = [rng.standard_normal((t, d)) for _, t in specs]
    packed = L.pack_adapters(adapters, inputs)
    w = rng.standard_normal((d, k)) / 8
    ups = [rng.standard_normal((t, k)) for _, t in specs]
    p = O.pack([a.down for a in adapters], [a.up for a in adapters], [a.alpha for a in adapters], inputs)
    ys, ref_y = L.packed_forward(packed, w), O.packed_forward(p, w)
    dd, du, dx = L.packed_backward(packed, w, ups)
    rd, ru, rx = O.packed_backward(p, w, ups)
    for i in range(len(specs)):
        close(ys[i], ref_y[i], f"y[{i}]")
        close(dd[i], rd[i], f"dA[{i}]")
        close(du[i], ru[i], f"dB[{i}]")
        close(dx[i], rx[i], f"dX[{i}]")
    assert ys[1].shape == (0, k) and not np.any(dd[1]) and not np.any(du[1])


def test_grad_check_small_pack():
    rng = np.random.default_rng(13)
    adapters = [L.AdapterWeights(rng.standard_normal((6, r)), rng.standard_normal((r, 5)),
                                 float(rng.uniform(0.2, 2.0))) for r in (1, 2, 3, 4)]
    inputs = [rng.standard_normal((int(rng.integers(1, 5)), 6)) for _ in adapters]
    report = L.grad_check(L.pack_adapters(adapters, inputs), rng.standard_normal((6, 5)), seed=99)
    assert set(report.case_errors) == {"up_weight", "up_input", "down_weight", "down_input"}
    assert report.passed, report.case_errors
