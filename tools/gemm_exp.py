"""GEMM experiment: TF/s of ops.gemm for a list of shapes under the current
PLORA_DEBUG_FLAGS / PLORA_* env (run once per variant; prints one JSON line).
Median over `reps` launches, L2 flushed before each, 3 passes over the shape list."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops  # noqa: E402

bf = torch.bfloat16
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
shapes = [(32768, 4096, 4096), (32768, 4096, 14336), (32768, 14336, 4096), (32768, 1024, 4096),
          (32768, 4096, 1024)]
ops_ = {}
for M, N, K in shapes:
    ops_[(M, N, K)] = (torch.randn(M, K, device="cuda").to(bf), torch.randn(N, K, device="cuda").to(bf))
res = {k: [] for k in ops_}
for _ in range(3):
    for (M, N, K), (a, w) in ops_.items():
        for _ in range(3):
            ops.gemm(a, w, True)
        for _ in range(int(os.environ.get("REPS", "8"))):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            ops.gemm(a, w, True)
            e.record()
            torch.cuda.synchronize()
            res[(M, N, K)].append(2 * M * N * K / s.elapsed_time(e) / 1e9)
out = {"flags": os.environ.get("PLORA_DEBUG_FLAGS", "0"), "tag": os.environ.get("TAG", "")}
for (M, N, K), v in res.items():
    out[f"{M}x{N}x{K}"] = round(statistics.median(v), 1)
print(json.dumps(out), flush=True)
