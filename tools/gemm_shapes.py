"""Time our GEMM on the in-step shapes (CUDA events, L2 flushed), optional residual."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2508_02932_b200 import ops
bf = torch.bfloat16
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, reps=8):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        flush.zero_(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts)//2]
for (M, N, K, kmaj, res) in [(32768, 4096, 4096, True, False), (32768, 4096, 4096, True, True), (32768, 4096, 1024, False, True),
                             (32768, 14336, 4096, True, False), (32768, 4096, 14336, True, True)]:
    a = torch.randn(M, K, device="cuda").to(bf)
    w = (torch.randn(N, K, device="cuda") if kmaj else torch.randn(K, N, device="cuda")).to(bf)
    r = torch.randn(M, N, device="cuda").to(bf) if res else None
    out = torch.empty(M, N, device="cuda", dtype=bf)
    ms = t(lambda: ops.gemm(a, w, kmaj, out=out, residual=r))
    print(f"M{M} N{N} K{K} {'k' if kmaj else 'mn'} res={res}: {2*M*N*K/ms/1e9:.0f} TF/s", flush=True)
