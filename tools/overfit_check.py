"""Full-size training sanity check: the C3 packed job (Llama-3.1-8B shapes, 16 adapters,
T = 32768) trained for N steps on ONE fixed synthetic batch.  Every adapter sees the same
batch each step, so a working forward / backward / per-adapter AdamW drives each adapter's
loss down at a speed set by its learning rate (2e-5 .. 4e-4).  Prints per-adapter losses.
  python tools/overfit_check.py [--steps 40]"""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--config", default="llama-3.1-8b")
args = ap.parse_args()
specs, s = bench_adapters(args.config)
tr = PackedLoraTrainer(PRESETS[args.config], specs, s, device="cuda")
tokens = tr.synthetic_tokens().cuda()
hist = []
for i in range(args.steps):
    hist.append(tr.step(tokens).float().cpu())
torch.cuda.synchronize()
print("adapter  rank  alpha   lr       loss@0    loss@mid  loss@end  change")
for a, sp in enumerate(specs):
    l0, lm, le = hist[0][a].item(), hist[len(hist) // 2][a].item(), hist[-1][a].item()
    print(f"{a:7d} {sp.rank:5d} {sp.alpha:6.1f} {sp.lr:.0e}  {l0:8.4f}  {lm:8.4f}  {le:8.4f}  {le - l0:+.4f}")
dec = sum(1 for a in range(len(specs)) if hist[-1][a] < hist[0][a])
print(f"{dec}/{len(specs)} adapters lower after {args.steps} steps; "
      f"finite: {all(torch.isfinite(h).all().item() for h in hist)}")
