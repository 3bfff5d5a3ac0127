"""One GEMM each: ours (pair or 1-CTA per PLORA_GEMM_PAIR) and cuBLAS, for ncu comparison."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2508_02932_b200 import ops
M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 8192, 8192)))
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
for _ in range(2):
    ops.gemm(a, w, True)
    a @ w.t()
torch.cuda.synchronize()
