"""torch.profiler breakdown of one C4 TP=8 rank-0 shard step (16 layers, collectives skipped)."""
import dataclasses
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from c4_shard_bench import NullComm  # noqa: E402
from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters  # noqa: E402

cfg = dataclasses.replace(PRESETS["qwen2.5-32b"], n_layers=16)
specs, s = bench_adapters("qwen2.5-32b")
tr = PackedLoraTrainer(cfg, specs, s, device="cuda", tp=NullComm(0, 8))
tok = tr.synthetic_tokens().cuda()
for _ in range(2):
    tr.step(tok)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tr.step(tok)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
