"""One packed-LoRA linear fwd+bwd at a C3 shape (for ncu launch lists / captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops  # noqa: E402
from paper_2508_02932_b200.meta import build_meta  # noqa: E402

bf = torch.bfloat16
d = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ranks = [8, 16, 32, 64] * 4
b = [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]
meta = build_meta(ranks, [x * 1024 for x in b], [r * m for r, m in zip(ranks, [0.25, 1, 2, 4] * 4)]).to("cuda")
T = meta.total_tokens
x = torch.randn(T, d, device="cuda").to(bf)
w = (torch.randn(k, d, device="cuda") * 0.02).to(bf)
a_sh = (torch.randn(16, d, 64, device="cuda") * 0.01).to(bf)
bt_sh = (torch.randn(16, k, 64, device="cuda") * 0.01).to(bf)
hs = torch.empty(T, 64, device="cuda", dtype=bf)
y = torch.empty(T, k, device="cuda", dtype=bf)
dy = torch.randn(T, k, device="cuda").to(bf)
dx = torch.empty(T, d, device="cuda", dtype=bf)
dh = torch.empty(T, 64, device="cuda", dtype=bf)
ga = torch.empty(d * meta.rpad16_total, device="cuda")
gb = torch.empty(k * meta.rpad16_total, device="cuda")
for _ in range(reps):
    ops.linear_fwd(meta, x, w, True, a_sh, bt_sh, hs, y)
    ops.linear_bwd(meta, x, w, True, a_sh, bt_sh, hs, dy, ga, gb, dx, True, dh)
torch.cuda.synchronize()
print("done")
