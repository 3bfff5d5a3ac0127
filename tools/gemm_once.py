"""Each GEMM shape launched twice (warm-up + measured) for ncu A/B captures
(ncu --clock-control base gives clock-stable per-launch durations)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops  # noqa: E402

bf = torch.bfloat16
shapes = [(32768, 4096, 4096), (32768, 4096, 14336), (32768, 14336, 4096), (32768, 1024, 4096),
          (32768, 4096, 1024)]
for M, N, K in shapes:
    a = torch.randn(M, K, device="cuda").to(bf)
    w = torch.randn(N, K, device="cuda").to(bf)
    for _ in range(2):
        ops.gemm(a, w, True)
    torch.cuda.synchronize()
    del a, w
