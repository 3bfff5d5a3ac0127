"""GPU counterpart of the reference's `lorasweep verify-kernels` (cli.py:187-262): runs
the drop-in packed-LoRA operators (paper_2508_02932_b200.lorapack, libplora on the
B200) on seeded random packs and prints the same five PASS/FAIL lines.

  packed-vs-sequential : packed_forward / packed_backward vs adapter_forward /
                         adapter_backward of every adapter alone (same pack shapes as
                         the reference harness); bf16-tier bound, relative to the
                         largest reference magnitude (the reference's own bound is
                         1e-12 / 1e-10 in float64)
  case 1..4            : dB, dH, dA, dX (dH from the K4 kernel, the rest from
                         packed_backward) vs the reference formulas (lorapack.py:219-230)
                         in float64 on the bf16-rounded operands, with the device's bf16
                         roundings of Hs and dH (max error over max(|ref|, 1); bound
                         GRAD_TOL).  The reference checks these cases by central
                         differences; through a bf16 forward those are dominated by the
                         rounding of the perturbed Hs / y (5-15% on these draws), so the
                         finite-difference check stays in the pytest suite (grad_check).

Exit code 7 (the reference's EXIT_VERIFY) on failure.
  python tools/verify_kernels.py [--seed 0] [--trials 64]
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_02932_b200 import lorapack as L  # noqa: E402

EXIT_VERIFY = 7
SEQ_TOL = 2e-2
GRAD_TOL = 1e-2


def _dh_error(adapters, ups, bf) -> float:
    """Case 2: dH_i = alpha_i dY_i B_i^T from the K4 kernel (plora_lora_shrink over the
    stacked B_i^T operand) vs float64 on the bf16 operands."""
    import torch

    from paper_2508_02932_b200 import ops
    from paper_2508_02932_b200.meta import build_meta

    ranks = [a.rank for a in adapters]
    meta = build_meta(ranks, [u.shape[0] for u in ups], [a.alpha for a in adapters]).to("cuda")
    k = ups[0].shape[1]
    kp = (k + 7) // 8 * 8
    bt = torch.zeros((len(adapters), kp, meta.rpad64), dtype=torch.bfloat16, device="cuda")
    for i, a in enumerate(adapters):
        bt[i, :k, :a.rank] = torch.from_numpy(a.up.T.copy()).to(torch.bfloat16)
    dy = torch.zeros((meta.total_tokens, kp), dtype=torch.bfloat16, device="cuda")
    dy[:, :k] = torch.from_numpy(np.concatenate(ups)).to(torch.bfloat16)
    dh = torch.empty((meta.total_tokens, meta.rpad64), dtype=torch.bfloat16, device="cuda")
    ops.shrink(meta, dy, bt, dh)
    got = dh.double().cpu().numpy()
    worst = 0.0
    for i, (a, u) in enumerate(zip(adapters, ups)):
        s0, s1 = meta.row_offsets[i], meta.row_offsets[i + 1]
        want = bf(a.alpha * (bf(u) @ bf(a.up).T))
        worst = max(worst, float(np.abs(got[s0:s1, :a.rank] - want).max() / max(np.abs(want).max(), 1.0)))
    return worst


def verify(seed: int, trials: int):
    rng = np.random.default_rng(seed)
    lines, ok = [], True
    worst_fwd = worst_bwd = 0.0
    for _ in range(trials):
        n = int(rng.integers(1, 9))
        d = 8 * int(rng.integers(1, 5))       # kernel dims are multiples of 8 (the reference draws 2..16)
        k = 8 * int(rng.integers(1, 5))
        adapters, inputs, ups = [], [], []
        for _ in range(n):
            r = int(rng.integers(1, 7))
            tokens = int(rng.integers(1, 7))
            adapters.append(L.AdapterWeights(down=rng.standard_normal((d, r)), up=rng.standard_normal((r, k)),
                                             alpha=float(rng.uniform(0.1, 2.0))))
            inputs.append(rng.standard_normal((tokens, d)))
            ups.append(rng.standard_normal((tokens, k)))
        w_base = rng.standard_normal((d, k))
        packed = L.pack_adapters(adapters, inputs)
        outs = L.packed_forward(packed, w_base)
        d_downs, d_ups, d_inputs = L.packed_backward(packed, w_base, ups)
        for i, (a, x, dy) in enumerate(zip(adapters, inputs, ups)):
            ref = L.adapter_forward(a, x, w_base)
            worst_fwd = max(worst_fwd, float(np.abs(outs[i] - ref).max() / max(np.abs(ref).max(), 1e-30)))
            rd, ru, rx = L.adapter_backward(a, x, w_base, dy)
            for got, want in ((d_downs[i], rd), (d_ups[i], ru), (d_inputs[i], rx)):
                worst_bwd = max(worst_bwd, float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-30)))
    seq_ok = worst_fwd < SEQ_TOL and worst_bwd < SEQ_TOL
    ok &= seq_ok
    lines.append(f"packed-vs-sequential  {'PASS' if seq_ok else 'FAIL'}   "
                 f"fwd {worst_fwd:.3e}  bwd {worst_bwd:.3e}  ({trials} packs)")
    # cases 1, 3, 4: the device gradients vs the reference formulas (lorapack.py:219-230)
    # evaluated in float64 on the bf16-rounded operands the device used; case 2 (dH, an
    # internal intermediate) by central differences through the device path (grad_check).
    def bf(a):
        import torch
        return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).double().numpy()

    worst = {"up_weight": 0.0, "up_input": 0.0, "down_weight": 0.0, "down_input": 0.0}
    for i in range(max(8, trials // 8)):
        n = int(rng.integers(1, 5))
        d = 8 * int(rng.integers(1, 3))
        k = 8 * int(rng.integers(1, 3))
        adapters, inputs, ups = [], [], []
        for _ in range(n):
            r = int(rng.integers(1, 5))
            tokens = int(rng.integers(1, 5))
            adapters.append(L.AdapterWeights(down=rng.standard_normal((d, r)), up=rng.standard_normal((r, k)),
                                             alpha=float(rng.uniform(0.1, 2.0))))
            inputs.append(rng.standard_normal((tokens, d)))
            ups.append(rng.standard_normal((tokens, k)))
        w = rng.standard_normal((d, k))
        packed = L.pack_adapters(adapters, inputs)
        dd, du, dx = L.packed_backward(packed, w, ups)
        for j, (a, x, dy) in enumerate(zip(adapters, inputs, ups)):
            A, B, X, DY, W = bf(a.down), bf(a.up), bf(x), bf(dy), bf(w)
            H = bf(a.alpha * (X @ A))                 # the device stores Hs = alpha X A in bf16
            DH = bf(a.alpha * (DY @ B.T))             # and dH = alpha dY B^T in bf16
            for key, got, want in (("up_weight", du[j], H.T @ DY), ("down_weight", dd[j], X.T @ DH),
                                   ("down_input", dx[j], DY @ W.T + DH @ A.T)):
                scale = max(np.abs(want).max(), 1.0)
                worst[key] = max(worst[key], float(np.abs(got - want).max() / scale))
        worst["up_input"] = max(worst["up_input"], _dh_error(adapters, ups, bf))
    names = {"up_weight": "case 1: up-projection weight grad", "up_input": "case 2: up-projection input grad",
             "down_weight": "case 3: down-projection weight grad", "down_input": "case 4: down-projection input grad"}
    for key, label in names.items():
        case_ok = worst[key] < GRAD_TOL
        ok &= case_ok
        lines.append(f"{label:38s}{'PASS' if case_ok else 'FAIL'}   max rel err {worst[key]:.3e}")
    return ok, lines


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--trials", type=int, default=64)
    args = ap.parse_args()
    ok, lines = verify(args.seed, args.trials)
    for line in lines:
        print(line)
    if not ok:
        print("error: verification: packed-adapter math check failed", file=sys.stderr)
        sys.exit(EXIT_VERIFY)


if __name__ == "__main__":
    main()
