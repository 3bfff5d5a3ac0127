"""C4 (Qwen2.5-32B, 32 packed adapters, TP = 8) on ONE B200: times one tensor-parallel
rank's shard of the step with the collectives replaced by local copies (sequence
parallelism on: the rank's token shard of the residual stream, full-T column/row GEMMs).
The shard is timed at two depths (default 32 and the full 64 layers) and the per-layer
time is their slope (every layer is identical work; lm_head / embedding / optimizer are
the intercept).

This is a COMPUTE-ONLY projection (the pool has one GPU, so the NCCL all-reduces of
a real TP=8 job cannot run here): every GEMM / LoRA / attention / optimizer kernel of
rank 0's shard runs at its real size, the all-reduces are skipped (so the numbers are
not those of the unsharded model).  Output: one JSON line with the rank's step time,
the job's projected tokens/s if communication were fully hidden, and the per-GPU
base-GEMM TF/s.  Usage: python tools/c4_shard_bench.py [--tp 8] [--steps 3] [--warmup 2]
"""
import argparse
import dataclasses
import json
import os
import sys

sys.path.insert(0, ".")
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402

from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters  # noqa: E402
from paper_2508_02932_b200.tp import Comm  # noqa: E402


class NullComm(Comm):
    """Rank `rank` of a `world`-rank group whose collectives are skipped (timing only)."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def all_reduce_(self, t, op="sum"):
        return t

    def all_gather_(self, out, inp):
        out[self.rank * inp.shape[0]:(self.rank + 1) * inp.shape[0]].copy_(inp)   # own rows; others stale
        return out

    def reduce_scatter_(self, out, inp):
        out.copy_(inp[self.rank * out.shape[0]:(self.rank + 1) * out.shape[0]])
        return out

    def reduce_(self, t, root):
        return t

    def broadcast_(self, t, root):
        return t


TRAINER_KW = {}


def time_shard(cfg, specs, s, tp, steps, warmup, graph=True):
    tr = PackedLoraTrainer(cfg, specs, s, device="cuda", tp=NullComm(0, tp), **TRAINER_KW)
    tokens = tr.synthetic_tokens().cuda()
    for _ in range(warmup):
        tr.step(tokens)
    torch.cuda.synchronize()
    run = tr.graphed(tokens, warmup=1).step if graph else (lambda: tr.step(tokens))   # as bench.py
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    out = (e0.elapsed_time(e1) / steps, tr.T, torch.cuda.max_memory_allocated() / 1e9, tr.save_normed)
    del tr, tokens
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--depths", default="32,64")
    ap.add_argument("--eager", action="store_true", help="time the eager step (default: the CUDA-graph step)")
    ap.add_argument("--no-fuse-dual", action="store_true")
    ap.add_argument("--no-fuse-swiglu-bwd", action="store_true")
    args = ap.parse_args()
    if args.no_fuse_dual:
        TRAINER_KW["fuse_dual"] = False
    if args.no_fuse_swiglu_bwd:
        TRAINER_KW["fuse_swiglu_bwd"] = False
    full = PRESETS["qwen2.5-32b"]
    specs, s = bench_adapters("qwen2.5-32b")
    depths = [int(x) for x in args.depths.split(",")]
    meas = {}
    for L in depths:
        meas[L] = time_shard(dataclasses.replace(full, n_layers=L), specs, s, args.tp, args.steps, args.warmup,
                             graph=not args.eager)
    if full.n_layers in meas:   # the full depth was measured: use it
        ms, T = meas[full.n_layers][0], meas[full.n_layers][1]
        per_layer = ms / full.n_layers
    else:                       # extrapolate from two depths (every layer is identical work)
        (l0, (m0, T, mem0, sn0)), (l1, (m1, _, mem1, sn1)) = sorted(meas.items())[:2]
        per_layer = (m1 - m0) / (l1 - l0)
        ms = m0 + per_layer * (full.n_layers - l0)
    cfg = full
    per_gpu_flops = cfg.base_flops_per_token() * T / args.tp
    ar_bytes = 4 * T * cfg.d * 2 * cfg.n_layers     # o + down fwd, qkv + gate/up bwd input grads (bf16)
    print(json.dumps({
        "workload": f"C4 {cfg.name}, {len(specs)} adapters, T={T}, rank 0 shard of TP={args.tp}",
        "kind": "compute-only projection: collectives skipped (1-GPU pool); not a bench value",
        "ms_per_step_rank": round(ms, 1),
        "job_tokens_per_s_if_comm_hidden": round(T / (ms / 1000.0), 1),
        "per_gpu_tokens_per_s_if_comm_hidden": round(T / (ms / 1000.0) / args.tp, 1),
        "per_gpu_base_gemm_tflops": round(per_gpu_flops / (ms / 1000.0) / 1e12, 1),
        "allreduce_bytes_per_rank_per_step": ar_bytes,
        "allreduce_ms_at_725GBps_busbw": round(ar_bytes * 2 * (args.tp - 1) / args.tp / 725e9 * 1000.0, 1),
        "measured": {str(L): {"ms_per_step": round(v[0], 1), "mem_peak_gb": round(v[2], 1), "save_normed": v[3]}
                     for L, v in meas.items()},
        "ms_per_layer": round(per_layer, 2),
        "step_mode": "eager" if args.eager else "cuda_graph",
        "trainer_options": TRAINER_KW,
    }), flush=True)


if __name__ == "__main__":
    main()
