"""Generate golden vectors by running the REAL reference (lorasweep) in this container.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Writes tests/golden/lorapack_golden.npz.  The reference cannot travel to the GPU
box (/root/reference is absent there), so the vectors are committed as small
fixtures and the GPU parity tests read them instead of importing lorasweep.

Cases (all inputs seeded, float64):
  * ``rp{j}``  -- random packs in the shape family of the reference's own
                  random_pack (pkg/tests/test_lorapack.py:16-25) and acceptance
                  criterion 1 (pkg/tests/test_acceptance.py:165-201)
  * ``edge{j}`` -- an empty token segment, rank 1, negative alpha, alpha = 0
  * ``lin{j}`` -- per-linear shapes of the bench configs at reduced token counts
                  (C1 tiny d=256 q/k/v/o/gate/up/down; a C3-like 4096 slice)
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/pkg/src")
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

import lorasweep  # noqa: E402  (the unmodified reference)
from lorasweep import AdapterWeights, pack_adapters, packed_backward, packed_forward  # noqa: E402


def _f32(a):
    """Round to float32-representable values so inputs can be stored losslessly as f32."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def _case(store: dict, name: str, downs, ups, alphas, inputs, w, dys):
    downs, ups, inputs, dys, w = ([_f32(a) for a in downs], [_f32(a) for a in ups],
                                  [_f32(a) for a in inputs], [_f32(a) for a in dys], _f32(w))
    adapters = [AdapterWeights(down=a, up=b, alpha=float(al)) for a, b, al in zip(downs, ups, alphas)]
    packed = pack_adapters(adapters, inputs)
    outs = packed_forward(packed, w)
    dd, du, dx = packed_backward(packed, w, dys)
    n = len(adapters)
    store[f"{name}/n"] = np.array(n)
    store[f"{name}/alphas"] = np.array(alphas, dtype=np.float64)
    store[f"{name}/rank_offsets"] = np.array(packed.rank_offsets, dtype=np.int64)
    store[f"{name}/row_offsets"] = np.array(packed.row_offsets, dtype=np.int64)
    store[f"{name}/w"] = w.astype(np.float32)
    store[f"{name}/down_block"] = packed.down_block.astype(np.float32)
    store[f"{name}/up_block"] = packed.up_block.astype(np.float32)
    store[f"{name}/inputs"] = packed.inputs.astype(np.float32)
    store[f"{name}/upstream"] = np.concatenate(dys, axis=0).astype(np.float32)
    store[f"{name}/y"] = np.concatenate(outs, axis=0)
    store[f"{name}/d_down"] = np.concatenate(dd, axis=1)
    store[f"{name}/d_up"] = np.concatenate(du, axis=0)
    store[f"{name}/d_input"] = np.concatenate(dx, axis=0)


def main() -> None:
    store: dict = {}
    rng = np.random.default_rng(20250804)
    names = []
    # random desk-scale packs (reference test family)
    for j in range(12):
        n = int(rng.integers(1, 9))
        d = int(rng.integers(2, 33))
        k = int(rng.integers(2, 33))
        downs, ups, alphas, inputs, dys = [], [], [], [], []
        for _ in range(n):
            r = int(rng.integers(1, 17))
            t = int(rng.integers(1, 9))
            downs.append(rng.standard_normal((d, r)))
            ups.append(rng.standard_normal((r, k)))
            alphas.append(float(rng.uniform(0.1, 2.0)))
            inputs.append(rng.standard_normal((t, d)))
            dys.append(rng.standard_normal((t, k)))
        _case(store, f"rp{j}", downs, ups, alphas, inputs, rng.standard_normal((d, k)), dys)
        names.append(f"rp{j}")
    # edge cases: empty segment, rank 1, negative / zero alpha, rank > 64
    d, k = 40, 24
    specs = [(3, 5, 1.5), (1, 0, 0.7), (16, 7, -0.8), (5, 4, 0.0), (70, 3, 0.3)]
    downs = [rng.standard_normal((d, r)) for r, _, _ in specs]
    ups = [rng.standard_normal((r, k)) for r, _, _ in specs]
    inputs = [rng.standard_normal((t, d)) for _, t, _ in specs]
    dys = [rng.standard_normal((t, k)) for _, t, _ in specs]
    _case(store, "edge0", downs, ups, [a for _, _, a in specs], inputs, rng.standard_normal((d, k)), dys)
    names.append("edge0")
    # per-linear shapes at bench-like sizes, reduced token counts (bf16-representable scales)
    lin_shapes = [(256, 256, [8, 16, 32, 64], [16, 32, 16, 32]),      # C1 q/o
                  (256, 512, [8, 16, 32, 64], [16, 32, 16, 32]),      # C1 gate/up-like (k > d)
                  (512, 256, [8, 16, 32, 64], [16, 32, 16, 32]),      # C1 down-like (d > k)
                  (128, 128, [8, 64, 16, 32, 8], [200, 64, 130, 1, 90])]  # multi-tile, unaligned
    for j, (d, k, ranks, toks) in enumerate(lin_shapes):
        mults = [0.25, 1.0, 2.0, 4.0]
        downs = [rng.uniform(-1, 1, (d, r)) / np.sqrt(d) for r in ranks]
        ups = [rng.standard_normal((r, k)) * 0.02 for r in ranks]
        alphas = [r * mults[i % 4] for i, r in enumerate(ranks)]
        inputs = [rng.standard_normal((t, d)) for t in toks]
        dys = [rng.standard_normal((t, k)) * 0.1 for t in toks]
        w = rng.standard_normal((d, k)) * 0.02
        _case(store, f"lin{j}", downs, ups, alphas, inputs, w, dys)
        names.append(f"lin{j}")
    store["__cases__"] = np.array(names)
    store["__reference_version__"] = np.array(lorasweep.__version__)
    out = ROOT / "tests" / "golden" / "lorapack_golden.npz"
    out.parent.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(out, **store)
    print(f"wrote {out} ({out.stat().st_size / 1e6:.2f} MB, {len(names)} cases)")


if __name__ == "__main__":
    main()
