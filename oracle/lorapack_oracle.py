"""ORACLE -- test infrastructure only.  Not part of the product path.

A float64 numpy restatement of the reference's packed multi-adapter LoRA
arithmetic (``lorasweep.lorapack``, /root/reference/pkg/src/lorasweep/lorapack.py).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``--impl reference`` / ``cpu_baseline``) may import this module, and only as the
checker or as the timed CPU reference -- never as a fallback for the GPU path.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by running the real reference
(``oracle/gen_golden.py`` -> ``tests/golden/lorapack_golden.npz``) and against
the literal known-answer values in the reference's own tests
(pkg/tests/test_lorapack.py:29-46, 70-74, 129-136).

Semantics kept exactly:
  * y_i = x_i W + alpha_i (x_i A_i) B_i with raw alpha (lorapack.py:8, 167-169)
  * rank/row offsets are Python-int prefix sums (lorapack.py:146-150)
  * Cases 1-4 of the backward (lorapack.py:18-21, 172-180, 219-230)
"""

from __future__ import annotations

from typing import Sequence

import numpy as np


def prefix_offsets(sizes: Sequence[int]) -> tuple[int, ...]:
    """Exact integer prefix sums starting at 0 (lorapack.py:146-150)."""
    out = [0]
    for s in sizes:
        out.append(out[-1] + int(s))
    return tuple(out)


def pack(downs: Sequence[np.ndarray], ups: Sequence[np.ndarray], alphas: Sequence[float],
         inputs: Sequence[np.ndarray]) -> dict:
    """Concatenate adapters and their token slices (lorapack.py:128-158).

    Returns a dict with the same content as the reference PackedAdapters:
    down_block (d x R), up_block (R x k), inputs (T x d), alphas, rank_offsets,
    row_offsets."""
    if len(downs) == 0:
        raise ValueError("nothing to pack")
    ranks = [a.shape[1] for a in downs]
    for a, b in zip(downs, ups):
        if a.shape[1] != b.shape[0]:
            raise ValueError("rank mismatch")
    return {
        "down_block": np.concatenate(list(downs), axis=1),
        "up_block": np.concatenate(list(ups), axis=0),
        "inputs": np.concatenate(list(inputs), axis=0),
        "alphas": tuple(float(a) for a in alphas),
        "rank_offsets": prefix_offsets(ranks),
        "row_offsets": prefix_offsets([x.shape[0] for x in inputs]),
    }


def token_adapter_ids(row_offsets: Sequence[int]) -> np.ndarray:
    """Per-token adapter id: np.repeat(arange(n), diff(row_offsets))."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    return np.repeat(np.arange(len(ro) - 1, dtype=np.int32), np.diff(ro))


def single_forward(down: np.ndarray, up: np.ndarray, alpha: float, x: np.ndarray,
                   w: np.ndarray) -> np.ndarray:
    """x W + alpha (x A) B (lorapack.py:167-169)."""
    return x @ w + alpha * ((x @ down) @ up)


def single_backward(down, up, alpha, x, w, dy):
    """(d_down, d_up, d_input) for one adapter (lorapack.py:172-180)."""
    h = x @ down
    d_up = alpha * (h.T @ dy)            # Case 1
    d_h = alpha * (dy @ up.T)            # Case 2
    d_down = x.T @ d_h                   # Case 3
    d_x = dy @ w.T + d_h @ down.T        # Case 4 (+ base path)
    return d_down, d_up, d_x


def packed_forward(p: dict, w: np.ndarray) -> list[np.ndarray]:
    """Packed forward over ragged segments (lorapack.py:183-199): one base GEMM
    over all tokens, then per segment the adapter's own low-rank path."""
    ro, so = p["rank_offsets"], p["row_offsets"]
    X = p["inputs"]
    base = X @ w
    outs = []
    for i, alpha in enumerate(p["alphas"]):
        rows = slice(so[i], so[i + 1])
        cols = slice(ro[i], ro[i + 1])
        h = X[rows] @ p["down_block"][:, cols]
        outs.append(base[rows] + alpha * (h @ p["up_block"][cols, :]))
    return outs


def packed_backward(p: dict, w: np.ndarray, dys: Sequence[np.ndarray]):
    """Packed backward (lorapack.py:202-231): returns (d_downs, d_ups, d_inputs)."""
    ro, so = p["rank_offsets"], p["row_offsets"]
    X = p["inputs"]
    dY = np.concatenate(list(dys), axis=0)
    dx_base = dY @ w.T
    d_downs, d_ups, d_inputs = [], [], []
    for i, alpha in enumerate(p["alphas"]):
        rows = slice(so[i], so[i + 1])
        cols = slice(ro[i], ro[i + 1])
        A = p["down_block"][:, cols]
        B = p["up_block"][cols, :]
        x, dy = X[rows], dY[rows]
        h = x @ A
        d_h = alpha * (dy @ B.T)
        d_ups.append(alpha * (h.T @ dy))
        d_downs.append(x.T @ d_h)
        d_inputs.append(dx_base[rows] + d_h @ A.T)
    return d_downs, d_ups, d_inputs


def rel_frobenius(got: np.ndarray, ref: np.ndarray) -> float:
    """||got - ref||_F / max(||ref||_F, tiny): the bf16-tier parity metric."""
    num = float(np.linalg.norm(np.asarray(got, np.float64) - np.asarray(ref, np.float64)))
    den = float(np.linalg.norm(np.asarray(ref, np.float64)))
    return num / max(den, 1e-30)


def max_abs_over_max_ref(got: np.ndarray, ref: np.ndarray) -> float:
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(np.asarray(got, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))
