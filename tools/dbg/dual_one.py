"""One fused K3+K4 (lora_dual) launch at the C3 pack for ncu (warm-up launches first).
  python tools/dbg/dual_one.py K [sep]"""
import sys, torch
sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta
bf = torch.bfloat16
K = int(sys.argv[1])
sep = len(sys.argv) > 2 and sys.argv[2] == "sep"
ranks = [8, 16, 32, 64] * 4
tokens = [x * 1024 for x in [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]]
meta = build_meta(ranks, tokens, [1.0] * len(ranks)).to("cuda")
T, R64 = meta.total_tokens, meta.rpad64
dy = torch.randn(T, K, device="cuda").to(bf)
bt = (torch.randn(len(ranks), K, R64, device="cuda") * 0.01).to(bf)
hs = (torch.randn(T, R64, device="cuda") * 0.1).to(bf)
dh = torch.empty(T, R64, device="cuda", dtype=bf)
g = torch.empty(K * meta.rpad16_total, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.sum()
    if sep:
        ops.shrink(meta, dy, bt, dh); ops.segred(meta, dy, hs, g)
    else:
        ops.lora_dual(meta, dy, bt, hs, dh, g)
torch.cuda.synchronize()
