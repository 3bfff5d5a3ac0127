"""Eager step vs CUDA-graph replay of the whole packed training step (C3)."""
import os
import sys
import time
sys.path.insert(0, ".")
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch
from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters

name = sys.argv[1] if len(sys.argv) > 1 else "llama-3.1-8b"
specs, s = bench_adapters(name)
tr = PackedLoraTrainer(PRESETS[name], specs, s, device="cuda")
tok = tr.synthetic_tokens().cuda()
for _ in range(3):
    tr.step(tok)
torch.cuda.synchronize()
def timed(fn, n=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
t_eager = timed(lambda: tr.step(tok))
h0 = time.perf_counter(); tr.step(tok); h1 = time.perf_counter(); torch.cuda.synchronize(); h2 = time.perf_counter()
print(f"eager {t_eager:.1f} ms/step; host enqueue {1000*(h1-h0):.1f} ms, drain {1000*(h2-h1):.1f} ms", flush=True)
g = torch.cuda.CUDAGraph()
s_ = torch.cuda.Stream()
s_.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s_):
    tr.step(tok)
torch.cuda.current_stream().wait_stream(s_)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    tr.step(tok)
torch.cuda.synchronize()
t_graph = timed(lambda: g.replay())
print(f"graph {t_graph:.1f} ms/step  mem {torch.cuda.max_memory_allocated()/1e9:.1f} GB", flush=True)
