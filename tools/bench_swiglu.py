"""Time the gate/up + SwiGLU pair GEMM (C3 shape) and the other in-step GEMM shapes
(CUDA events, L2 flushed with a read).  PLORA_LIB selects the library (A/B)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta
bf = torch.bfloat16
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, reps=10):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        flush.sum(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts)//2]
ranks = [8, 16, 32, 64] * 4
tokens = [x * 1024 for x in [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]]
meta = build_meta(ranks, tokens, [float(r) for r in ranks]).to("cuda")
T, d, f = meta.total_tokens, 4096, 14336
x = torch.randn(T, d, device="cuda").to(bf)
wg = (torch.randn(f, d, device="cuda") * 0.02).to(bf); wu = (torch.randn(f, d, device="cuda") * 0.02).to(bf)
btg = (torch.randn(16, f, 64, device="cuda") * 0.02).to(bf); btu = (torch.randn(16, f, 64, device="cuda") * 0.02).to(bf)
hsg = (torch.randn(T, 64, device="cuda")).to(bf); hsu = (torch.randn(T, 64, device="cuda")).to(bf)
fl = 2 * 2 * T * d * f
ms = t(lambda: ops.linear_gate_up_swiglu(meta, x, wg, wu, btg, btu, hsg, hsu))
print(f"gate/up+swiglu T{T} d{d} f{f}: {ms*1e3:.0f} us  {fl/ms/1e9:.0f} TF/s", flush=True)
del wg, wu, btg, btu
for (M, N, K, kmaj) in [(32768, 4096, 4096, True), (32768, 4096, 14336, True), (32768, 14336, 4096, False), (4096, 4096, 4096, True)]:
    a = torch.randn(M, K, device="cuda").to(bf)
    w = (torch.randn(N, K, device="cuda") if kmaj else torch.randn(K, N, device="cuda")).to(bf)
    out = torch.empty(M, N, device="cuda", dtype=bf)
    ms = t(lambda: ops.gemm(a, w, kmaj, out=out))
    print(f"gemm M{M} N{N} K{K} {'k' if kmaj else 'mn'}: {ms*1e3:.0f} us {2*M*N*K/ms/1e9:.0f} TF/s", flush=True)
