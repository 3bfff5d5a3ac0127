"""One shrink / segred launch at a chosen pack for ncu (warm-up launches first)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta
bf = torch.bfloat16
pack, K, mode = sys.argv[1], int(sys.argv[2]), sys.argv[3]
ranks, tokens = {"c3": ([8, 16, 32, 64] * 4, [x * 1024 for x in [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]]),
                 "split8": ([64], [4096])}[pack]
meta = build_meta(ranks, tokens, [1.0] * len(ranks)).to("cuda")
if mode == "whole":
    def whole(m):
        s = m.struct; s.d_ws = None; s.ws_bytes = 0; return s
    ops._pack = whole
T, R64 = meta.total_tokens, meta.rpad64
p = torch.randn(T, K, device="cuda").to(bf)
l_sh = (torch.randn(len(ranks), K, R64, device="cuda") * 0.01).to(bf)
q = (torch.randn(T, R64, device="cuda") * 0.1).to(bf)
hs = torch.empty(T, R64, device="cuda", dtype=bf)
g = torch.empty(K * meta.rpad16_total, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.sum(); ops.shrink(meta, p, l_sh, hs); flush.sum(); ops.segred(meta, p, q, g)
torch.cuda.synchronize()
