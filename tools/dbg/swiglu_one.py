"""One fused SwiGLU-backward + dA launch at the C3 shape for ncu (warm-up launches first)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta
bf = torch.bfloat16
ranks = [8, 16, 32, 64] * 4
tokens = [x * 1024 for x in [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]]
meta = build_meta(ranks, tokens, [1.0] * len(ranks)).to("cuda")
T, F = meta.total_tokens, 14336
da = (torch.randn(T, F, device="cuda") * 0.1).to(bf)
g = torch.randn(T, F, device="cuda").to(bf)
u = torch.randn(T, F, device="cuda").to(bf)
dh = (torch.randn(T, meta.rpad64, device="cuda") * 0.1).to(bf)
ga = torch.empty(F * meta.rpad16_total, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.sum()
    ops.swiglu_bwd_segred(meta, da, g, u, dh, ga)
torch.cuda.synchronize()
