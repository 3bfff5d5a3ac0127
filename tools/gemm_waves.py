"""Pair-GEMM tile width vs wave quantisation: time the base GEMM on the in-step shapes at the
planner-split token counts (T = 32768 / n_gpus) with CUDA events, L2 flushed between runs.
Run once per libplora build (PLORA_LIB=...) to compare tile policies."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2508_02932_b200 import ops
bf = torch.bfloat16
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


tag = sys.argv[1] if len(sys.argv) > 1 else "lib"
for T in (4096, 8192, 16384, 32768):
    for (N, K, kmaj) in [(14336, 4096, False), (14336, 4096, True), (4096, 14336, True), (4096, 4096, True)]:
        a = torch.randn(T, K, device="cuda").to(bf)
        w = (torch.randn(N, K, device="cuda") if kmaj else torch.randn(K, N, device="cuda")).to(bf)
        out = torch.empty(T, N, device="cuda", dtype=bf)
        ms = t(lambda: ops.gemm(a, w, kmaj, out=out))
        print(f"{tag} T{T} N{N} K{K} {'k' if kmaj else 'mn'}: {ms * 1e3:.1f} us {2 * T * N * K / ms / 1e9:.0f} TF/s",
              flush=True)
        del a, w, out
