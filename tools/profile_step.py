"""torch.profiler breakdown of one packed training step (C3 by default)."""
import sys
sys.path.insert(0, ".")
import os
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch
from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters

name = sys.argv[1] if len(sys.argv) > 1 else "llama-3.1-8b"
specs, s = bench_adapters(name)
tr = PackedLoraTrainer(PRESETS[name], specs, s, device="cuda")
tok = tr.synthetic_tokens().cuda()
for _ in range(2):
    tr.step(tok)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    tr.step(tok)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=45, max_name_column_width=90))
