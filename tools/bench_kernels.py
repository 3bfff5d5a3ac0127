"""Kernel micro-benchmarks (CUDA events, warmed, L2 flushed between reps):
tcgen05 GEMM vs torch.matmul (cuBLAS) and the packed-LoRA linear fwd/bwd at C3 shapes."""

import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops  # noqa: E402
from paper_2508_02932_b200.meta import build_meta  # noqa: E402

bf = torch.bfloat16
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


res = {}
for (M, N, K) in [(8192, 8192, 8192), (32768, 4096, 4096), (32768, 14336, 4096), (32768, 4096, 14336),
                  (32768, 1024, 4096)]:
    a = torch.randn(M, K, device="cuda").to(bf)
    w = torch.randn(N, K, device="cuda").to(bf)
    fl = 2 * M * N * K
    t_ours = timeit(lambda: ops.gemm(a, w, True))
    t_ours_mn = timeit(lambda: ops.gemm(a, w.t().contiguous() if False else w, True))
    wt = w.t().contiguous()
    t_mn = timeit(lambda: ops.gemm(a, wt, False))
    t_cublas = timeit(lambda: a @ w.t())
    res[f"gemm_{M}x{N}x{K}"] = {"ours_kmajor_tflops": fl / t_ours / 1e9, "ours_mnmajor_tflops": fl / t_mn / 1e9,
                                "cublas_tflops": fl / t_cublas / 1e9}
    print(f"GEMM {M}x{N}x{K}: ours(K-major B) {fl / t_ours / 1e9:.0f} TF/s  ours(MN-major B) "
          f"{fl / t_mn / 1e9:.0f} TF/s  cuBLAS {fl / t_cublas / 1e9:.0f} TF/s", flush=True)
    del a, w, wt

# packed linear at C3: 16 adapters, T=32768, q-proj 4096x4096
ranks = [8, 16, 32, 64] * 4
b = [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]
tokens = [x * 1024 for x in b]
alphas = [r * m for r, m in zip(ranks, [0.25, 1, 2, 4] * 4)]
meta = build_meta(ranks, tokens, alphas).to("cuda")
T = meta.total_tokens
for d, k in [(4096, 4096), (4096, 14336), (14336, 4096)]:
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
    t_f = timeit(lambda: ops.linear_fwd(meta, x, w, True, a_sh, bt_sh, hs, y))
    t_b = timeit(lambda: ops.linear_bwd(meta, x, w, True, a_sh, bt_sh, hs, dy, ga, gb, dx, True, dh))
    t_base = timeit(lambda: ops.gemm(x, w, True, y))
    fl = 2 * T * d * k
    print(f"linear {d}x{k}: fwd {t_f:.3f} ms ({fl / t_f / 1e9:.0f} TF/s base-equiv), bwd {t_b:.3f} ms "
          f"({fl / t_b / 1e9:.0f}), base GEMM alone {t_base:.3f} ms", flush=True)
    res[f"linear_{d}x{k}"] = {"fwd_ms": t_f, "bwd_ms": t_b, "base_gemm_ms": t_base}
    del x, w, y, dy, dx
print(json.dumps(res))
