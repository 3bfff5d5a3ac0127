"""Fixed per-launch cost of the LoRA kernels inside a CUDA graph: 64 back-to-back launches
of a one-tile problem (T = 128 tokens) replayed, vs a trivial torch kernel and vs the real
T = 4096 problem.  Prints us per launch."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta
bf = torch.bfloat16


def per_launch(fn, n=64, reps=5):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1000 / n)
    return best


x = torch.zeros(16, device="cuda")
print("torch add_ (1 block)        %.2f us" % per_launch(lambda: x.add_(1)))
for T in (128, 4096):
    meta = build_meta([64], [T], [1.0]).to("cuda")
    K = 4096
    p = torch.randn(T, K, device="cuda").to(bf)
    l_sh = (torch.randn(1, K, 64, device="cuda") * 0.01).to(bf)
    q = (torch.randn(T, 64, device="cuda") * 0.1).to(bf)
    hs = torch.empty(T, 64, device="cuda", dtype=bf)
    g = torch.empty(K * meta.rpad16_total, device="cuda")
    dh = torch.empty(T, 64, device="cuda", dtype=bf)
    print(f"T={T:5d} shrink             %.2f us" % per_launch(lambda: ops.shrink(meta, p, l_sh, hs)))
    print(f"T={T:5d} segred             %.2f us" % per_launch(lambda: ops.segred(meta, p, q, g)))
    print(f"T={T:5d} dual (K4+K3)       %.2f us" % per_launch(lambda: ops.lora_dual(meta, p, l_sh, q, dh, g)))
